// The whole CG loop of solve_least_squares (src/lsq.cpp:88-107) as ONE persistent
// cooperative kernel, for problems whose A is L2-resident (BASELINE c1, c2).
//
// The multi-kernel loop (k_pcg.cu: pass, reduce, upd1, upd2 per iteration, host poll every 4)
// costs ~37 us per iteration at c1 and ~55 us at c2 in launch gaps and polls, against a
// 1 MiB / 64 MiB pass.  Here every iteration is four phases separated by grid barriers:
//
//   P  pass      each CTA streams its column block of A once: t_j = (A^H w)_j, s_c += A_j t_j,
//                the lagged r / x updates, and (qq, Re<r,t>, ||r||^2) partials  (= pcg_pass_kernel)
//   R  reduce    CTA c sums rows [c*rs, (c+1)*rs) of s over the CTA partials in fixed order;
//                every CTA sums the scalar partials (same order, same result) -> alpha = gg/qq
//   U1 gradient  CTA c owns the same row slice: g_j -= alpha (Rinv^H s)_j, u_j += alpha dir_j,
//                ax_j += alpha s_j, dir_old_j = dir_j, ||g_slice||^2               (= pcg_upd1_kernel)
//   U2 direction every CTA sums ||g||^2 (fixed order), runs the stop test of lsq.cpp:101 on its
//                replicated CgState copy (all CTAs decide identically), then
//                dir = g + beta dir_old and w_i = (Rinv dir)_i for its slice     (= pcg_upd2_kernel)
//
// The arithmetic of every phase is that of the multi-kernel path (same formulas, FMA forms and
// stop rule); only the order of the partial sums differs (CTA partials of a different grid), so
// iterates agree to rounding, and the result is bitwise reproducible run to run.  The CgState
// lives in shared memory in every CTA (identical copies); CTA 0 writes it back at the end.
#include <cooperative_groups.h>

#include <algorithm>

#include "pcg.cuh"

namespace mnb {

namespace {

namespace cg = cooperative_groups;

constexpr int kMaxWarps = 16;

__device__ __forceinline__ double2 warp_sum2s(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

// Fixed-order warp sums over the G CTA partials: lane l adds parts l, l+32, ... in order, then a
// fixed xor butterfly (deterministic; 32 loads in flight instead of a G-long dependent chain).
__device__ __forceinline__ double warp_sum_parts(const double* base, int stride, int G, int lane) {
    double acc = 0.0;
    for (int b = lane; b < G; b += 32) acc += __ldcg(base + int64_t(b) * stride);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc;
}
__device__ __forceinline__ double2 warp_sum_parts2(const double2* base, int64_t stride, int G, int lane) {
    double2 acc = make_double2(0.0, 0.0);
    for (int b = lane; b < G; b += 32) acc = c_add(acc, __ldcg(base + int64_t(b) * stride));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    return acc;
}

template <typename AT>
__device__ __forceinline__ AT ldA(const void* A, int64_t idx);
template <>
__device__ __forceinline__ double2 ldA<double2>(const void* A, int64_t idx) {
    return __ldcg(static_cast<const double2*>(A) + idx);
}
template <>
__device__ __forceinline__ double ldA<double>(const void* A, int64_t idx) {
    return __ldcg(static_cast<const double*>(A) + idx);
}

__device__ __forceinline__ void dot_accs(double2& acc, double2 a, double2 w) {  // conj(a) w
    acc.x = fma(a.x, w.x, fma(a.y, w.y, acc.x));
    acc.y = fma(a.x, w.y, fma(-a.y, w.x, acc.y));
}
__device__ __forceinline__ void dot_accs(double2& acc, double a, double2 w) {
    acc.x = fma(a, w.x, acc.x);
    acc.y = fma(a, w.y, acc.y);
}
__device__ __forceinline__ void axpy_accs(double2& acc, double2 a, double2 t) {  // a t
    acc.x = fma(a.x, t.x, fma(-a.y, t.y, acc.x));
    acc.y = fma(a.x, t.y, fma(a.y, t.x, acc.y));
}
__device__ __forceinline__ void axpy_accs(double2& acc, double a, double2 t) {
    acc.x = fma(a, t.x, acc.x);
    acc.y = fma(a, t.y, acc.y);
}

// Phases R, U1, U2 of one CG iteration (see the header) over `parts` pass partials; every CTA
// keeps the same CgState copy S.  Returns true when the loop stops (the state says why).
template <int W>
__device__ bool cg_update(const SmallCgArgs& p, int parts, CgState& S, double2* v_sh, double (*red_sh)[4],
                          cg::grid_group& grid) {
    const int64_t m = p.m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x, G = gridDim.x;
    const int64_t rs = (m + G - 1) / G, r0 = ::min(m, int64_t(c) * rs), r1 = ::min(m, r0 + rs);
        // ------------------------------------------------------------ R: reduce
        // (parts == 0: already reduced -- the distributed loop's allreduced [s | qq, rt, rr] in p.s)
        if (parts > 0) {
            for (int64_t i = r0 + warp; i < r1; i += W) {  // a warp per row of the slice
                const double2 acc = warp_sum_parts2(p.part_s + i, m, parts, lane);
                if (lane == 0) p.s[i] = acc;
            }
            if (warp < 3) {  // a warp per scalar (every CTA: identical sums)
                const double acc = warp_sum_parts(p.part_scal + warp, 4, parts, lane);
                if (lane == 0) red_sh[0][warp] = acc;
            }
        } else if (threadIdx.x < 3) {
            red_sh[0][threadIdx.x] = __ldcg(reinterpret_cast<const double*>(p.s) + 2 * m + threadIdx.x);
        }
        __syncthreads();
        const double qq_t = red_sh[0][0], rt_t = red_sh[0][1], rrk = red_sh[0][2];
        if (qq_t == 0.0) {  // lsq.cpp:91: break before any update
            if (threadIdx.x == 0) {
                S.done = 1;
                S.stop_qq0 = 1;
                S.alpha = 0.0;
                S.rr = rrk;
                if (c == 0) p.residual_norms[S.iterations] = sqrt(rrk);
            }
            __syncthreads();
            return true;
        }
        const double alpha = S.gg / qq_t;
        grid.sync();
        // ---------------------------------------------------------- U1: gradient
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) v_sh[i] = __ldcg(p.s + i);
        __syncthreads();
        double my = 0.0;
        for (int64_t j = r0 + warp; j < r1; j += W) {
            const double2* col = p.Rinv + j * m;  // column j of Rinv: entries i <= j
            double2 acc = make_double2(0.0, 0.0);
            for (int64_t i = lane; i <= j; i += 32) {
                const double2 a = __ldcg(col + i), b = v_sh[i];
                acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));  // conj(a) b
                acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
            }
            acc = warp_sum2s(acc);
            if (lane == 0) {
                if (p.ax) {
                    double2 axj = p.ax[j];
                    axj.x = fma(alpha, v_sh[j].x, axj.x);
                    axj.y = fma(alpha, v_sh[j].y, axj.y);
                    p.ax[j] = axj;
                }
                const double2 dj = p.dir[j];
                double2 uj = p.u[j];
                uj.x = fma(alpha, dj.x, uj.x);
                uj.y = fma(alpha, dj.y, uj.y);
                p.u[j] = uj;
                p.dir_old[j] = dj;
                double2 gj = p.g[j];
                gj.x = fma(-alpha, acc.x, gj.x);
                gj.y = fma(-alpha, acc.y, gj.y);
                p.g[j] = gj;
                my += gj.x * gj.x + gj.y * gj.y;
            }
        }
        if (lane == 0) red_sh[warp][3] = my;
        __syncthreads();
        if (threadIdx.x == 0) {
            double acc = 0.0;
            for (int q = 0; q < W; ++q) acc += red_sh[q][3];
            p.part_gg[c] = acc;
            // replicated state (pcg_upd1_kernel's block-0 epilogue)
            if (c == 0) p.residual_norms[S.iterations] = sqrt(rrk);
            S.rr = rrk - 2.0 * alpha * rt_t + alpha * alpha * qq_t;
            S.alpha = alpha;
            S.iterations += 1;
            S.gg_prev = S.gg;
        }
        grid.sync();
        // --------------------------------------------------------- U2: direction
        if (warp == 0) {
            const double ggn = warp_sum_parts(p.part_gg, 1, gridDim.x, lane);  // fixed order, every CTA
            if (lane == 0) {
            const double excess = S.dup * ggn;
            const bool conv = excess <= S.tau * fmax(S.rr - excess, 0.0) || S.rr <= S.floor2;
            const bool capped = S.iterations >= S.max_iterations;
            S.excess = excess;
            if (conv || capped || ggn == 0.0) {
                S.done = 1;
                S.converged = conv ? 1 : 0;
                S.gg = ggn;
            } else {
                red_sh[0][3] = ggn / S.gg_prev;  // beta
                S.gg = ggn;
            }
            }
        }
        __syncthreads();
        if (S.done) return true;
        const double beta = red_sh[0][3];
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
            const double2 gi = __ldcg(p.g + i), di = __ldcg(p.dir_old + i);
            v_sh[i] = make_double2(fma(beta, di.x, gi.x), fma(beta, di.y, gi.y));
        }
        __syncthreads();
        for (int64_t i = r0 + warp; i < r1; i += W) {
            const double2* row = p.Rinv_rows + i * m;  // row i of Rinv: entries j >= i
            double2 acc = make_double2(0.0, 0.0);
            for (int64_t jj = i + lane; jj < m; jj += 32) {
                const double2 a = __ldcg(row + jj), b = v_sh[jj];
                acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
                acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
            }
            acc = warp_sum2s(acc);
            if (lane == 0) {
                p.w[i] = acc;
                p.dir[i] = v_sh[i];
            }
        }
        return false;
}

// One CG iteration's m-space work for the multi-kernel loop (A too large for L2): the phases above
// in one cooperative launch after each fused pass, instead of the reduce / upd1 / upd2 kernels
// (k_pcg.cu).  State in global memory (read by the pass, written back by CTA 0).
template <int W>
__global__ void __launch_bounds__(W * 32, 1) pcg_update_kernel(const SmallCgArgs p, int parts) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double2 sm[];
    __shared__ double red_sh[kMaxWarps][4];
    __shared__ CgState S;
    if (threadIdx.x == 0) S = *p.st;
    __syncthreads();
    if (S.done) return;  // uniform: every CTA read the same state
    cg_update<W>(p, parts, S, sm, red_sh, grid);
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.st = S;
}

// EPL: rows per lane (m <= 32 EPL).  Shared memory: w / s / d (m each), the per-warp s partials
// [kSmallWarps][m], scalar scratch.
// W warps per CTA: 16, or 8 at EPL >= 4 (more registers per thread: no spills)
template <typename AT, int EPL, int W>
__global__ void __launch_bounds__(W * 32, 1) pcg_small_kernel(const SmallCgArgs p) {
    constexpr int kSmallWarps = W;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double2 sm[];
    const int64_t m = p.m, n = p.n;
    double2* w_sh = sm;                 // m
    double2* v_sh = sm + m;             // m: s (U1) / d (U2)
    double2* wp = sm + 2 * m;           // [warps][m]
    __shared__ double red_sh[kMaxWarps][4];
    __shared__ CgState S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, c = blockIdx.x;
    if (threadIdx.x == 0) S = *p.st;
    __syncthreads();
    // this CTA's column block (its row slice of the m-space phases is taken in cg_update)
    const int64_t per = (n + G - 1) / G, c0 = ::min(n, int64_t(c) * per), c1 = ::min(n, c0 + per);

    while (!S.done) {
        // ------------------------------------------------------------- P: pass
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) w_sh[i] = __ldcg(p.w + i);
        __syncthreads();
        const double alpha_prev = S.alpha;
        double2 sacc[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) sacc[e] = make_double2(0.0, 0.0);
        double qq = 0.0, rt = 0.0, rr = 0.0;
        // the r / t / x entries of the warp's first 32 columns, prefetched one per lane (the
        // per-column epilogue then takes them by shuffle instead of a dependent global load)
        double2 pt = make_double2(0.0, 0.0), pr = pt, px = pt;
        {
            const int64_t jl = c0 + 2 * warp + 2 * int64_t(kSmallWarps) * (lane >> 1) + (lane & 1);
            if (jl < c1) {
                pt = p.t[jl];
                pr = p.r[jl];
                if (p.x) px = p.x[jl];
            }
        }
        int step = 0;
        // two columns per step: their loads and reductions are independent (latency hiding)
        for (int64_t j0 = c0 + 2 * warp; j0 < c1; j0 += 2 * kSmallWarps, ++step) {
            double2 told_s, r_s, x_s;
            {
                const int src = (2 * step + (lane & 1)) & 31;
                told_s = make_double2(__shfl_sync(0xffffffffu, pt.x, src), __shfl_sync(0xffffffffu, pt.y, src));
                r_s = make_double2(__shfl_sync(0xffffffffu, pr.x, src), __shfl_sync(0xffffffffu, pr.y, src));
                x_s = make_double2(__shfl_sync(0xffffffffu, px.x, src), __shfl_sync(0xffffffffu, px.y, src));
            }
            const int nk = j0 + 1 < c1 ? 2 : 1;
            AT a[2][EPL];
            double2 dacc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    const int64_t row = lane + 32 * e;
                    if (row < m && k < nk) {
                        a[k][e] = ldA<AT>(p.A, (j0 + k) * m + row);
                        dot_accs(dacc[k], a[k][e], w_sh[row]);
                    } else {
                        a[k][e] = AT{};
                    }
                }
            double2 tks[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) tks[k] = warp_sum2s(dacc[k]);
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    if (lane + 32 * e < m) axpy_accs(sacc[e], a[k][e], tks[k]);
            if (lane < nk) {  // the lagged updates of column j (pcg_pass_kernel's epilogue, PCG_CG)
                const int64_t j = j0 + lane;
                const double2 tk = lane == 0 ? tks[0] : tks[1];
                const bool pre = step < 16;
                const double2 told = pre ? told_s : p.t[j];
                double2 rk = pre ? r_s : p.r[j];
                rk.x = fma(-alpha_prev, told.x, rk.x);
                rk.y = fma(-alpha_prev, told.y, rk.y);
                rr = fma(rk.x, rk.x, fma(rk.y, rk.y, rr));
                rt = fma(rk.x, tk.x, fma(rk.y, tk.y, rt));
                p.r[j] = rk;
                p.t[j] = tk;
                if (p.x) {
                    double2 xk = pre ? x_s : p.x[j];
                    xk.x = fma(alpha_prev, told.x, xk.x);
                    xk.y = fma(alpha_prev, told.y, xk.y);
                    p.x[j] = xk;
                }
                qq = fma(tk.x, tk.x, fma(tk.y, tk.y, qq));
            }
        }
        // lanes 0 and 1 hold the column scalars: fixed-order combine into lane 0
        qq += __shfl_down_sync(0xffffffffu, qq, 1);
        rt += __shfl_down_sync(0xffffffffu, rt, 1);
        rr += __shfl_down_sync(0xffffffffu, rr, 1);
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            const int64_t row = lane + 32 * e;
            if (row < m) wp[int64_t(warp) * m + row] = sacc[e];
        }
        if (lane == 0) {
            red_sh[warp][0] = qq;
            red_sh[warp][1] = rt;
            red_sh[warp][2] = rr;
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
            double2 acc = wp[i];
            for (int q = 1; q < kSmallWarps; ++q) acc = c_add(acc, wp[int64_t(q) * m + i]);
            p.part_s[int64_t(c) * m + i] = acc;
        }
        if (threadIdx.x < 3) {
            double acc = 0.0;
            for (int q = 0; q < kSmallWarps; ++q) acc += red_sh[q][threadIdx.x];
            p.part_scal[c * 4 + threadIdx.x] = acc;
        }
        grid.sync();
        if (cg_update<W>(p, G, S, v_sh, red_sh, grid)) break;
        grid.sync();
    }
    if (c == 0 && threadIdx.x == 0) *p.st = S;
}

template <typename AT, int EPL>
void launch_small_typed(const SmallCgArgs& a, int grid, cudaStream_t stream) {
    constexpr int W = EPL >= 4 ? 8 : 16;
    auto k = pcg_small_kernel<AT, EPL, W>;
    const size_t smem = size_t(2 + W) * size_t(a.m) * 16;
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SmallCgArgs args = a;
    void* params[] = {&args};
    MNB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(W * 32), params,
                                         smem, stream));
}

template <int EPL>
void launch_small_epl(const SmallCgArgs& a, int grid, cudaStream_t stream) {
    if (a.is_real) launch_small_typed<double, EPL>(a, grid, stream);
    else launch_small_typed<double2, EPL>(a, grid, stream);
}

}  // namespace

int pcg_update_grid(int64_t m, int num_sms) {
    // one warp per row of a slice: rows / 8 CTAs of 8 warps, at most one CTA per SM
    return int(std::max<int64_t>(1, std::min<int64_t>(num_sms, (m + 7) / 8)));
}

void launch_pcg_update(const SmallCgArgs& a, int parts, int grid, cudaStream_t stream) {
    auto k = pcg_update_kernel<8>;
    const size_t smem = size_t(a.m) * 16;
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SmallCgArgs args = a;
    void* params[] = {&args, &parts};
    MNB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(8 * 32), params, smem,
                                         stream));
}

bool pcg_small_eligible(int64_t m, int64_t n, int is_real) {
    const size_t bytes = size_t(m) * size_t(n) * (is_real ? 8 : 16);
    return m >= 1 && m <= kSmallMaxM && bytes <= (size_t(96) << 20);  // A L2-resident
}

int pcg_small_grid(int64_t m, int64_t n, int num_sms) {
    // one CTA per 64 columns (4 per warp), at most one per SM
    const int64_t by_cols = (n + 63) / 64;
    return int(std::max<int64_t>(1, std::min<int64_t>(num_sms, std::max<int64_t>(by_cols, (m + 63) / 64))));
}

void launch_pcg_small(const SmallCgArgs& a, int grid, cudaStream_t stream) {
    const int epl = int((a.m + 31) / 32);
    if (epl <= 2) launch_small_epl<2>(a, grid, stream);
    else if (epl <= 4) launch_small_epl<4>(a, grid, stream);
    else launch_small_epl<8>(a, grid, stream);
}

}  // namespace mnb
