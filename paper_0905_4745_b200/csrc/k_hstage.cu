// H stage of the SRFT (src/srft.cpp:49-70): diagonal, permutation and the
// chain of n-1 plane rotations, applied to many rows at once.
//
// Data layout: a row block of `rows` rows of the (conj) matrix, column-major,
// element (r, k) at base[row0 + r + k*ld]; every column segment of a warp is
// 32 consecutive rows = 512 contiguous bytes.  All rows share the same
// parameters, so the operator acts on whole columns.
//
// The rotation chain (src/kernels_scalar.cpp:15-33) is a first-order linear
// recurrence in the carried value with real multiplier sin(theta_j)
// (SURVEY.md §0.4).  Each thread owns one row and one chunk of `chunk`
// columns and restarts the recurrence at a host-computed halo start past
// the chunk boundary, where the product of |sin| has decayed below 2^-70
// (host_srft.cpp: chain_halos) -- so the chunks run in parallel and the
// result matches the sequential chain to rounding.  Arithmetic uses the
// _rn intrinsics in the reference's operand order: with an exact carry the
// output is bit-identical to the reference scalar kernel.
#include "common.cuh"
#include "kernels.cuh"

namespace mnb {

namespace {

struct Fetch {
    const void* __restrict__ in;
    int in_real, in_conj;
    int64_t ld_in, in_row0;
    const int32_t* __restrict__ gather;
    const double2* __restrict__ in_diag;
    int in_diag_conj;
    int* nonfinite;

    __device__ __forceinline__ int64_t src_of(int64_t k) const { return gather ? int64_t(__ldg(gather + k)) : k; }
    __device__ __forceinline__ double2 load(int64_t r, int64_t src) const {
        const int64_t off = in_row0 + r + src * ld_in;
        double2 x;
        if (in_real) x = make_double2(__ldg(static_cast<const double*>(in) + off), 0.0);
        else x = __ldg(static_cast<const double2*>(in) + off);
        if (nonfinite && !(isfinite(x.x) && isfinite(x.y))) *nonfinite = 1;
        if (in_conj) x.y = -x.y;
        if (in_diag) {
            double2 dg = __ldg(in_diag + src);
            if (in_diag_conj) dg.y = -dg.y;
            x = c_mul_rn(x, dg);
        }
        return x;
    }
};

struct Emit {
    double2* __restrict__ out;
    int64_t ld_out, out_row0;
    const int32_t* __restrict__ scatter;
    const double2* __restrict__ out_diag;
    int out_diag_conj;
    __device__ __forceinline__ void store(int64_t r, int64_t o, double2 v) const {
        const int64_t dst = scatter ? int64_t(__ldg(scatter + o)) : o;
        if (out_diag) {
            double2 dg = __ldg(out_diag + dst);
            if (out_diag_conj) dg.y = -dg.y;
            v = c_mul_rn(v, dg);
        }
        out[out_row0 + r + dst * ld_out] = v;
    }
    // the same in two halves: destination index and diagonal entry fetched a batch ahead (two
    // dependent loads that would otherwise stall every step of the in-order recurrence loop:
    // ~1.4 us per step for a single row, 120 us per stage at any n)
    __device__ __forceinline__ void prefetch(int64_t o, int32_t& dst, double2& dg) const {
        dst = scatter ? __ldg(scatter + o) : int32_t(o);
        dg = make_double2(1.0, 0.0);
        if (out_diag) {
            dg = __ldg(out_diag + dst);
            if (out_diag_conj) dg.y = -dg.y;
        }
    }
    __device__ __forceinline__ void store_pre(int64_t r, int32_t dst, double2 dg, double2 v) const {
        if (out_diag) v = c_mul_rn(v, dg);
        out[out_row0 + r + int64_t(dst) * ld_out] = v;
    }
};

constexpr int kThreads = 128;
constexpr int kUnroll = 8;

// forward chain, rotation_chain_scalar(adjoint=false):
//   carry_j = cs_j x_j + sn_j carry_{j+1};  out_{j+1} = -sn_j x_j + cs_j carry_{j+1};  out_0 = carry_0
// adjoint chain, rotation_chain_scalar(adjoint=true):
//   out_j = cs_j carry_j - sn_j x_{j+1};    carry_{j+1} = sn_j carry_j + cs_j x_{j+1};  out_{n-1} = carry_{n-1}
__global__ void __launch_bounds__(kThreads) hstage_kernel(Fetch f, Emit e, const double2* __restrict__ cssn,
                                                          const int32_t* __restrict__ halo, int adjoint,
                                                          int64_t rows, int64_t n, int64_t chunk,
                                                          int64_t nchunks, int rows_per_cta) {
    const int t = threadIdx.x;
    const int64_t r = int64_t(blockIdx.x) * rows_per_cta + (t % rows_per_cta);
    const int64_t c = int64_t(blockIdx.y) * (kThreads / rows_per_cta) + (t / rows_per_cta);
    if (r >= rows || c >= nchunks) return;
    const int64_t i0 = c * chunk;
    const int64_t i1 = min(n, i0 + chunk);
    const int64_t start = __ldg(halo + c);

    if (!adjoint) {
        double2 carry = f.load(r, f.src_of(start));
        const int64_t lo = i0 > 0 ? i0 - 1 : 0;
        int64_t j = start - 1;
        // two batches in flight: the next batch's (index -> element) loads are issued before the
        // current batch's dependent recurrence runs (a single row is pure load latency otherwise)
        double2 x[kUnroll], cs[kUnroll], xn[kUnroll], csn[kUnroll], dg[kUnroll], dgn[kUnroll];
        int32_t dst[kUnroll], dstn[kUnroll];
        int cnt = 0;
        {
            const int64_t left = j - lo + 1;
            cnt = int(left < kUnroll ? (left > 0 ? left : 0) : kUnroll);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (u < cnt) {
                    x[u] = f.load(r, f.src_of(j - u));
                    cs[u] = __ldg(cssn + (j - u));
                    if (j - u + 1 < i1) e.prefetch(j - u + 1, dst[u], dg[u]);
                }
        }
        while (cnt > 0) {
            const int64_t jn = j - cnt;
            const int64_t leftn = jn - lo + 1;
            const int cntn = int(leftn < kUnroll ? (leftn > 0 ? leftn : 0) : kUnroll);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (u < cntn) {
                    xn[u] = f.load(r, f.src_of(jn - u));
                    csn[u] = __ldg(cssn + (jn - u));
                    if (jn - u + 1 < i1) e.prefetch(jn - u + 1, dstn[u], dgn[u]);
                }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (u < cnt) {
                    const double c_ = cs[u].x, s_ = cs[u].y;
                    const double2 a = x[u];
                    const double2 nc = make_double2(__dadd_rn(__dmul_rn(c_, a.x), __dmul_rn(s_, carry.x)),
                                                    __dadd_rn(__dmul_rn(c_, a.y), __dmul_rn(s_, carry.y)));
                    const double2 o = make_double2(__dadd_rn(__dmul_rn(-s_, a.x), __dmul_rn(c_, carry.x)),
                                                   __dadd_rn(__dmul_rn(-s_, a.y), __dmul_rn(c_, carry.y)));
                    if (j - u + 1 < i1) e.store_pre(r, dst[u], dg[u], o);
                    carry = nc;
                }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                x[u] = xn[u];
                cs[u] = csn[u];
                dst[u] = dstn[u];
                dg[u] = dgn[u];
            }
            j = jn;
            cnt = cntn;
        }
        if (i0 == 0) e.store(r, 0, carry);
    } else {
        double2 carry = f.load(r, f.src_of(start));
        const int64_t hi = min(i1, n - 1);
        int64_t j = start;
        double2 x[kUnroll], cs[kUnroll], xn[kUnroll], csn[kUnroll], dg[kUnroll], dgn[kUnroll];
        int32_t dst[kUnroll], dstn[kUnroll];
        int cnt = 0;
        {
            const int64_t left = hi - j;
            cnt = int(left < kUnroll ? (left > 0 ? left : 0) : kUnroll);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (u < cnt) {
                    x[u] = f.load(r, f.src_of(j + u + 1));
                    cs[u] = __ldg(cssn + (j + u));
                    if (j + u >= i0) e.prefetch(j + u, dst[u], dg[u]);
                }
        }
        while (cnt > 0) {
            const int64_t jn = j + cnt;
            const int64_t leftn = hi - jn;
            const int cntn = int(leftn < kUnroll ? (leftn > 0 ? leftn : 0) : kUnroll);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (u < cntn) {
                    xn[u] = f.load(r, f.src_of(jn + u + 1));
                    csn[u] = __ldg(cssn + (jn + u));
                    if (jn + u >= i0) e.prefetch(jn + u, dstn[u], dgn[u]);
                }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (u < cnt) {
                    const double c_ = cs[u].x, s_ = cs[u].y;
                    const double2 b = x[u];
                    const double2 o = make_double2(__dsub_rn(__dmul_rn(c_, carry.x), __dmul_rn(s_, b.x)),
                                                   __dsub_rn(__dmul_rn(c_, carry.y), __dmul_rn(s_, b.y)));
                    const double2 nc = make_double2(__dadd_rn(__dmul_rn(s_, carry.x), __dmul_rn(c_, b.x)),
                                                    __dadd_rn(__dmul_rn(s_, carry.y), __dmul_rn(c_, b.y)));
                    if (j + u >= i0) e.store_pre(r, dst[u], dg[u], o);
                    carry = nc;
                }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                x[u] = xn[u];
                cs[u] = csn[u];
                dst[u] = dstn[u];
                dg[u] = dgn[u];
            }
            j = jn;
            cnt = cntn;
        }
        if (i1 == n) e.store(r, n - 1, carry);
    }
}

}  // namespace

void launch_hstage(const HStageArgs& a, cudaStream_t stream) {
    Fetch f{a.in, a.in_real, a.in_conj, a.ld_in, a.in_row0, a.gather, a.in_diag, a.in_diag_conj, a.nonfinite};
    Emit e{a.out, a.ld_out, a.out_row0, a.scatter, a.out_diag, a.out_diag_conj};
    int rpc = 1;
    while (rpc < kThreads && rpc < a.rows) rpc <<= 1;
    const int chunks_per_cta = kThreads / rpc;
    dim3 grid(ceil_div(a.rows, rpc), ceil_div(a.nchunks, chunks_per_cta));
    require(grid.y <= 65535u, MNB_ERR_UNSUPPORTED, "hstage: too many chunks for one launch");
    hstage_kernel<<<grid, kThreads, 0, stream>>>(f, e, a.cssn, a.halo, a.adjoint, a.rows, a.n, a.chunk,
                                                 a.nchunks, rpc);
    MNB_LAUNCH_CHECK();
}

}  // namespace mnb
