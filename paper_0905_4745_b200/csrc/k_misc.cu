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

namespace mnb {

namespace {

// The CG's initial vectors without a pass over A (see launch_cg_init_vectors):
// r = c, t = 0, x = 0 and per-block partial sums of ||c||^2 (fixed order).
__global__ void __launch_bounds__(256) cg_init_vectors_kernel(const double2* __restrict__ c, int64_t n, double2* r,
                                                              double2* t, double2* x, double* part) {
    __shared__ double sh[8];
    double acc = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double2 v = c[i];
        r[i] = v;
        t[i] = make_double2(0.0, 0.0);
        if (x) x[i] = make_double2(0.0, 0.0);
        acc = fma(v.x, v.x, fma(v.y, v.y, acc));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) s += sh[w];
        part[blockIdx.x] = s;
    }
}

// y[j] = sum_i conj(S[i, j]) z[i] for the column-major l x m sketch: one CTA per column,
// fixed-order tree sum (deterministic).
__global__ void __launch_bounds__(256) sketch_adjoint_gemv_kernel(const double2* __restrict__ S, int64_t l,
                                                                  const double2* __restrict__ z, double2* y) {
    __shared__ double2 sh[8];
    const double2* col = S + int64_t(blockIdx.x) * l;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = threadIdx.x; i < l; i += blockDim.x) {
        const double2 a = col[i], b = z[i];
        acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
        acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 s = sh[0];
        for (int w = 1; w < int(blockDim.x >> 5); ++w) {
            s.x += sh[w].x;
            s.y += sh[w].y;
        }
        y[blockIdx.x] = s;
    }
}

// Power steps on D = Q1^H Q1 - I without host round trips (solver.cu cholqr_r): v <- v / ||v||
// and a copy into the work vector; then a <- a - v (= D v) and v <- a.
__global__ void unit_copy_kernel(double2* v, double2* a, int64_t m, const double* nrm) {
    const double s = 1.0 / *nrm;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        double2 x = v[i];
        x.x *= s;
        x.y *= s;
        v[i] = x;
        a[i] = x;
    }
}
__global__ void sub_copy_kernel(double2* a, double2* v, int64_t m) {
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const double2 d = make_double2(a[i].x - v[i].x, a[i].y - v[i].y);
        a[i] = d;
        v[i] = d;
    }
}

// red_scal = [qq = ||c||^2, <r,t> = 0, ||r||^2 = 0, 0] (the INIT pass's scalars, pcg.cuh)
__global__ void cg_init_finish_kernel(const double* part, int parts, double* red_scal) {
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += part[b];
    red_scal[0] = s;
    red_scal[1] = 0.0;
    red_scal[2] = 0.0;
    red_scal[3] = 0.0;
}

}  // namespace

void launch_unit_copy(double2* v, double2* a, int64_t m, const double* nrm, cudaStream_t stream) {
    unit_copy_kernel<<<1, 256, 0, stream>>>(v, a, m, nrm);
    MNB_LAUNCH_CHECK();
}

void launch_sub_copy(double2* a, double2* v, int64_t m, cudaStream_t stream) {
    sub_copy_kernel<<<1, 256, 0, stream>>>(a, v, m);
    MNB_LAUNCH_CHECK();
}

void launch_sketch_adjoint_gemv(const double2* S, int64_t l, int64_t m, const double2* z, double2* y,
                                cudaStream_t stream) {
    sketch_adjoint_gemv_kernel<<<unsigned(m), 256, 0, stream>>>(S, l, z, y);
    MNB_LAUNCH_CHECK();
}

void launch_cg_init_vectors(const double2* c, int64_t n, double2* r, double2* t, double2* x, double* part, int parts,
                            double* red_scal, cudaStream_t stream) {
    cg_init_vectors_kernel<<<parts, 256, 0, stream>>>(c, n, r, t, x, part);
    MNB_LAUNCH_CHECK();
    cg_init_finish_kernel<<<1, 1, 0, stream>>>(part, parts, red_scal);
    MNB_LAUNCH_CHECK();
}

}  // namespace mnb

namespace mnb {
namespace {
__global__ void conj_inplace_kernel(double2* x, int64_t count) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        x[i].y = -x[i].y;
}
}  // namespace

void launch_conj_inplace(double2* x, int64_t count, cudaStream_t stream) {
    if (count <= 0) return;
    conj_inplace_kernel<<<unsigned(std::min<int64_t>(ceil_div(count, 256), 148 * 16)), 256, 0, stream>>>(x, count);
    MNB_LAUNCH_CHECK();
}
}  // namespace mnb

namespace mnb {
namespace {
__global__ void real_to_complex_kernel(const double* in, double2* out, int64_t count) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = make_double2(in[i], 0.0);
}
}  // namespace

void launch_real_to_complex(const double* in, double2* out, int64_t count, cudaStream_t stream) {
    if (count <= 0) return;
    real_to_complex_kernel<<<unsigned(std::min<int64_t>(ceil_div(count, 256), 148 * 16)), 256, 0, stream>>>(in, out,
                                                                                                            count);
    MNB_LAUNCH_CHECK();
}
}  // namespace mnb
