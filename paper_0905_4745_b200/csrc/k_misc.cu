// Small glue kernels of the hot path.
#include "common.cuh"
#include "kernels.cuh"

namespace mnb {

namespace {

// with-replacement sampling: duplicate frequencies reuse the first slot's row.
__global__ void copy_dups_kernel(double2* S, int64_t ldS, int64_t row0, int64_t rows, const int32_t* dups,
                                 int64_t ndups) {
    const int64_t p = blockIdx.y;
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= ndups || r >= rows) return;
    const int64_t dst = dups[2 * p], src = dups[2 * p + 1];
    S[dst + (row0 + r) * ldS] = S[src + (row0 + r) * ldS];
}

// S^* v (src/srft.cpp:138-139): w = 0, w[sample[j]] += v[j].  Without
// replacement every target is distinct (parallel); with replacement the
// accumulation runs in the reference's j order on one thread.
__global__ void scatter_sample_kernel(const double2* v, int64_t l, const int32_t* sample, double2* w) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= l) return;
    const double2 x = v[j];
    w[sample[j]] = make_double2(0.0 + x.x, 0.0 + x.y);
}
__global__ void scatter_add_serial_kernel(const double2* v, int64_t l, const int32_t* sample, double2* w) {
    for (int64_t j = 0; j < l; ++j) {
        double2 a = w[sample[j]];
        a.x += v[j].x;
        a.y += v[j].y;
        w[sample[j]] = a;
    }
}

}  // namespace

void launch_copy_dups(double2* S, int64_t ldS, int64_t row0, int64_t rows, const int32_t* dups, int64_t ndups,
                      cudaStream_t stream) {
    if (ndups <= 0 || rows <= 0) return;
    require(ndups <= 65535, MNB_ERR_UNSUPPORTED, "too many duplicate samples");
    dim3 grid(ceil_div(rows, 128), unsigned(ndups));
    copy_dups_kernel<<<grid, 128, 0, stream>>>(S, ldS, row0, rows, dups, ndups);
    MNB_LAUNCH_CHECK();
}

void launch_scatter_add_sample(const double2* v, int64_t l, const int32_t* sample, int with_replacement, double2* w,
                               int64_t n, cudaStream_t stream) {
    MNB_CUDA(cudaMemsetAsync(w, 0, size_t(n) * sizeof(double2), stream));
    if (with_replacement) scatter_add_serial_kernel<<<1, 1, 0, stream>>>(v, l, sample, w);
    else scatter_sample_kernel<<<ceil_div(l, 256), 256, 0, stream>>>(v, l, sample, w);
    MNB_LAUNCH_CHECK();
}

}  // namespace mnb
