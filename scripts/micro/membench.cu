// Micro-benchmark: HBM bandwidth vs access-segment size and pattern on B200.
// Each warp moves one segment of SEG bytes per step (lanes read 16 B each,
// SEG/16 lanes active per segment, several segments per warp for SEG < 512).
// Patterns: 0 = contiguous, 1 = strided (segment k at k*stride), 2 = random permutation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void seg_copy(const double2* __restrict__ in, double2* __restrict__ out, const uint32_t* __restrict__ segs,
                         int64_t nseg, int seg16, int write) {
    const int sh = __ffs(seg16) - 1;
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t total = nseg * seg16;
    double2 acc = make_double2(0, 0);
    for (int64_t e = tid; e < total; e += nthreads) {
        const int64_t s = e >> sh, w = e & (seg16 - 1);
        const int64_t src = int64_t(segs[s]) * seg16 + w;
        if (write == 2) {  // scatter: contiguous read, segment-granular random write
            out[src] = __ldg(in + s * seg16 + w);
            continue;
        }
        double2 v = __ldg(in + src);
        if (write) out[s * seg16 + w] = v;
        else { acc.x += v.x; acc.y += v.y; }
    }
    if (!write && acc.x == 12345.678) out[0] = acc;
}

int main() {
    const int64_t bytes = int64_t(8) << 30;  // 8 GiB source
    const int64_t n16 = bytes / 16;
    double2 *in, *out;
    cudaMalloc(&in, bytes);
    cudaMalloc(&out, bytes);
    cudaMemset(in, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int seg : {64, 128, 256, 512}) {
        const int seg16 = seg / 16;
        const int64_t nseg = n16 / seg16;
        for (int pat = 0; pat < 3; ++pat) {
            std::vector<uint32_t> h(nseg);
            for (int64_t i = 0; i < nseg; ++i) h[i] = uint32_t(i);
            if (pat == 1) {  // stride: visit segments in transposed order of a 1024 x (nseg/1024) grid
                const int64_t rows = 1024, cols = nseg / rows;
                for (int64_t i = 0; i < nseg; ++i) h[i] = uint32_t((i % rows) * cols + i / rows);
            } else if (pat == 2) {
                std::mt19937_64 g(1);
                std::shuffle(h.begin(), h.end(), g);
            }
            uint32_t* d;
            cudaMalloc(&d, nseg * 4);
            cudaMemcpy(d, h.data(), nseg * 4, cudaMemcpyHostToDevice);
            for (int write = 0; write < 3; ++write) {
                seg_copy<<<sms * 8, 256>>>(in, out, d, nseg, seg16, write);
                cudaEventRecord(e0);
                const int reps = 3;
                for (int r = 0; r < reps; ++r) seg_copy<<<sms * 8, 256>>>(in, out, d, nseg, seg16, write);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double moved = double(bytes) * (write ? 2 : 1) + double(nseg) * 4;
                printf("{\"seg\": %d, \"pattern\": \"%s\", \"op\": \"%s\", \"GBps\": %.1f}\n", seg,
                       pat == 0 ? "contig" : pat == 1 ? "strided" : "random", write == 2 ? "scatter" : write ? "copy" : "read",
                       moved * reps / (ms * 1e-3) / 1e9);
            }
            cudaFree(d);
        }
    }
    return 0;
}
