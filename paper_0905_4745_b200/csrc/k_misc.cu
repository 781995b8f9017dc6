// Small glue kernels of the hot path.
#include <algorithm>

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

__global__ void zero_lower_kernel(double2* A, int64_t m) {
    const int64_t j = blockIdx.y;  // column
    for (int64_t i = j + 1 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
        A[i + j * m] = make_double2(0.0, 0.0);
}

void launch_zero_lower(double2* A, int64_t m, cudaStream_t stream) {
    if (m <= 1) return;
    dim3 grid(unsigned(std::min<int64_t>(16, ceil_div(m, 256))), unsigned(m));
    zero_lower_kernel<<<grid, 256, 0, stream>>>(A, m);
    MNB_LAUNCH_CHECK();
}

__global__ void max_offset_kernel(const double2* A, int64_t m, unsigned long long* out) {
    __shared__ double ws[8];
    double mx = 0.0;
    const int64_t total = m * m;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % m, j = e / m;
        if (i > j) continue;
        double2 a = A[e];
        if (i == j) a.x -= 1.0;
        mx = fmax(mx, fmax(fabs(a.x), fabs(a.y)));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) mx = fmax(mx, ws[w]);
        if (mx != mx) mx = 1e300;  // NaN: treat as not orthonormal
        atomicMax(out, __double_as_longlong(mx));  // non-negative doubles order like their bit patterns
    }
}

void launch_max_offset_from_identity(const double2* A, int64_t m, double* out, cudaStream_t stream) {
    MNB_CUDA(cudaMemsetAsync(out, 0, sizeof(double), stream));
    const int blocks = int(std::min<int64_t>(592, ceil_div(m * m, 256)));
    max_offset_kernel<<<blocks, 256, 0, stream>>>(A, m, reinterpret_cast<unsigned long long*>(out));
    MNB_LAUNCH_CHECK();
}

// Chain restart points for chunks of `chunk` indices (host_srft.cpp chain_halos,
// same 2^-70 rule) -- finer chunks than the operator's, for single vectors.
__global__ void chain_halo_kernel(const double2* __restrict__ cssn, int64_t n, int64_t chunk, int64_t nchunks,
                                  int32_t* fwd, int32_t* adj) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    constexpr double thr = 0x1.0p-70;
    const int64_t i0 = c * chunk, i1 = min(n, i0 + chunk);
    int64_t t = i1;
    if (i1 >= n) {
        t = n - 1;
    } else {
        double p = 1.0;
        while (t < n - 1 && p > thr) { p *= fabs(cssn[t].y); ++t; }
    }
    fwd[c] = int32_t(t);
    int64_t s = i0;
    double p = 1.0;
    while (s > 0 && p > thr) { --s; p *= fabs(cssn[s].y); }
    adj[c] = int32_t(s);
}

void launch_chain_halos(const double2* cssn, int64_t n, int64_t chunk, int64_t nchunks, int32_t* fwd, int32_t* adj,
                        cudaStream_t stream) {
    chain_halo_kernel<<<ceil_div(nchunks, 128), 128, 0, stream>>>(cssn, n, chunk, nchunks, fwd, adj);
    MNB_LAUNCH_CHECK();
}

__global__ void add_diagonal_kernel(double2* A, int64_t m, double shift) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < m) A[j + j * m].x += shift;
}

void launch_add_diagonal(double2* A, int64_t m, double shift, cudaStream_t stream) {
    add_diagonal_kernel<<<ceil_div(m, 256), 256, 0, stream>>>(A, m, shift);
    MNB_LAUNCH_CHECK();
}

}  // namespace mnb
