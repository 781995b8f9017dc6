// Fused preconditioned-CG pass and m-space updates (sm_100a).
//
// The reference spends each CG iteration of solve_least_squares on two GEMVs
// over B = A^H and two triangular solves (src/lsq.cpp:71-74,89-98).  Here one
// iteration is ONE streaming pass over A:
//     for every column k:  t_k = (A^H w)_k  (dot product down the column)
//                          s  += A[:,k] t_k  (axpy from the same registers)
// with w = R'^{-1} dir, so A is read from HBM exactly once per iteration; the
// gradient is carried by g <- g - alpha R'^{-H} s (since M^H q = R'^{-H} A t).
// The n-vector residual r is still materialised -- one iteration lagged, in
// the same pass -- so ||r||^2 is exact as in the reference (lsq.cpp:95).
//
// Pipeline: one CTA per SM; a producer warp streams column tiles of A (and the
// matching r / t segments) into a ring of shared-memory stages with
// cp.async.bulk (TMA bulk copies) completing on mbarriers; 16 consumer warps
// split each column's rows (G warps per column group) and reduce the dot
// product with shuffles + a named barrier.  Reductions are fixed-order, so
// results are bitwise reproducible run to run.
#include "pcg.cuh"

namespace mnb {

namespace {

constexpr int kConsumerWarps = 16;
constexpr int kThreads = (kConsumerWarps + 1) * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

template <typename AT>
__device__ __forceinline__ AT zero_of();
template <>
__device__ __forceinline__ double2 zero_of<double2>() { return make_double2(0.0, 0.0); }
template <>
__device__ __forceinline__ double zero_of<double>() { return 0.0; }

// conj(a) * w  accumulated into acc
template <typename AT>
__device__ __forceinline__ void dot_acc(double2& acc, AT a, double2 w);
template <>
__device__ __forceinline__ void dot_acc<double2>(double2& acc, double2 a, double2 w) {
    acc.x = fma(a.x, w.x, fma(a.y, w.y, acc.x));
    acc.y = fma(a.x, w.y, fma(-a.y, w.x, acc.y));
}
template <>
__device__ __forceinline__ void dot_acc<double>(double2& acc, double a, double2 w) {
    acc.x = fma(a, w.x, acc.x);
    acc.y = fma(a, w.y, acc.y);
}
// acc += a * t
template <typename AT>
__device__ __forceinline__ void axpy_acc(double2& acc, AT a, double2 t);
template <>
__device__ __forceinline__ void axpy_acc<double2>(double2& acc, double2 a, double2 t) {
    acc.x = fma(a.x, t.x, fma(-a.y, t.y, acc.x));
    acc.y = fma(a.x, t.y, fma(a.y, t.x, acc.y));
}
template <>
__device__ __forceinline__ void axpy_acc<double>(double2& acc, double a, double2 t) {
    acc.x = fma(a, t.x, acc.x);
    acc.y = fma(a, t.y, acc.y);
}

struct SmemLayout {
    size_t tileA, tileT, tileR, stage_bytes, red, bars, total;
};

__host__ __device__ inline SmemLayout smem_layout(int64_t m, int64_t C, int esz, int stages) {
    SmemLayout L;
    const size_t a = size_t(C) * size_t(m) * size_t(esz);
    L.tileA = 0;
    L.tileT = (a + 127) & ~size_t(127);
    L.tileR = L.tileT + ((size_t(C) * 16 + 127) & ~size_t(127));
    L.stage_bytes = L.tileR + ((size_t(C) * 16 + 127) & ~size_t(127));
    L.red = size_t(stages) * L.stage_bytes;                     // [8 groups][2 bufs][16 warps] complex
    L.bars = L.red + size_t(8 * 2 * kConsumerWarps) * 16;
    L.total = L.bars + size_t(2 * stages) * 8;
    return L;
}

template <typename AT, int EPL>
__global__ void __launch_bounds__(kThreads, 1) pcg_pass_kernel(const PcgPassArgs p, int G, int cpg, int stages,
                                                               int64_t C) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (p.state && p.state->done) return;  // uniform: converged loops cost one launch
    const int64_t m = p.m;
    const int esz = int(sizeof(AT));
    const SmemLayout L = smem_layout(m, C, esz, stages);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + stages;
    double2* red = reinterpret_cast<double2*>(smem + L.red);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NG = kConsumerWarps / G;
    // contiguous column range of this CTA
    const int64_t per = (p.n + gridDim.x - 1) / gridDim.x;
    const int64_t cb = min(p.n, int64_t(blockIdx.x) * per), ce = min(p.n, cb + per);
    const int64_t nstage = (ce - cb + C - 1) / C;
    const bool need_t = p.mode == PCG_INIT || p.mode == PCG_CG;
    const bool need_r = p.mode == PCG_CG;
    const double alpha_prev = (p.mode == PCG_CG && p.state) ? p.state->alpha : 0.0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kConsumerWarps) {
        // ------------------------------------------------------ producer
        if (lane == 0) {
            for (int64_t s = 0; s < nstage; ++s) {
                const int slot = int(s % stages);
                if (s >= stages) mbar_wait(&empty[slot], uint32_t(((s / stages) - 1) & 1));
                const int64_t c0 = cb + s * C;
                const int64_t cc = min(C, ce - c0);
                unsigned char* st = smem + slot * L.stage_bytes;
                const uint32_t abytes = uint32_t(cc * m * esz);
                const uint32_t vbytes = uint32_t(cc * 16);
                mbar_expect_tx(&full[slot], abytes + (need_t ? vbytes : 0u) + (need_r ? vbytes : 0u));
                bulk_g2s(st + L.tileA, static_cast<const unsigned char*>(p.A) + size_t(c0) * size_t(m) * esz, abytes,
                         &full[slot]);
                if (need_t) bulk_g2s(st + L.tileT, p.tin + c0, vbytes, &full[slot]);
                if (need_r) bulk_g2s(st + L.tileR, p.r + c0, vbytes, &full[slot]);
            }
        }
        // the producer warp joins the epilogue's block-wide barriers below
    }

    // ---------------------------------------------------------- consumers
    const int gq = warp / G, wig = warp % G;
    double2 wreg[EPL], sacc[EPL];
    const int row0 = wig * 32 + lane, rstep = 32 * G, mi = int(m);
#define ROW(e) (row0 + (e) * rstep)
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        sacc[e] = make_double2(0.0, 0.0);
        wreg[e] = make_double2(0.0, 0.0);
    }
    double qq = 0.0, rt = 0.0, rr = 0.0;  // leader-lane partials
    if (warp < kConsumerWarps) {
        if (p.mode != PCG_INIT) {
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (ROW(e) < mi) wreg[e] = p.w[ROW(e)];
        }
        int buf = 0;
        for (int64_t s = 0; s < nstage; ++s) {
            const int slot = int(s % stages);
            mbar_wait(&full[slot], uint32_t((s / stages) & 1));
            const int64_t c0 = cb + s * C;
            const int64_t cc = min(C, ce - c0);
            const unsigned char* st = smem + slot * L.stage_bytes;
            const AT* tA = reinterpret_cast<const AT*>(st + L.tileA);
            const double2* tT = reinterpret_cast<const double2*>(st + L.tileT);
            const double2* tR = reinterpret_cast<const double2*>(st + L.tileR);
            for (int i = 0; i < cpg; ++i) {
                const int64_t col = int64_t(gq) + int64_t(i) * NG;  // column within the stage
                if (col >= cc) break;                                 // uniform per group
                AT a[EPL];
#pragma unroll
                for (int e = 0; e < EPL; ++e) a[e] = ROW(e) < mi ? tA[int(col) * mi + ROW(e)] : zero_of<AT>();
                double2 t;
                if (p.mode == PCG_INIT) {
                    t = tT[col];
                } else {
                    double2 part = make_double2(0.0, 0.0);
#pragma unroll
                    for (int e = 0; e < EPL; ++e) dot_acc<AT>(part, a[e], wreg[e]);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double2 q = shfl_xor2(part, o);
                        part.x += q.x;
                        part.y += q.y;
                    }
                    if (G == 1) {
                        t = part;
                    } else {
                        double2* rb = red + (gq * 2 + buf) * kConsumerWarps;
                        if (lane == 0) rb[wig] = part;
                        named_bar(1 + gq, G * 32);
                        t = rb[0];
                        for (int k = 1; k < G; ++k) t = c_add(t, rb[k]);
                        buf ^= 1;
                    }
                }
#pragma unroll
                for (int e = 0; e < EPL; ++e) axpy_acc<AT>(sacc[e], a[e], t);
                if (wig == 0 && lane == 0) {
                    const int64_t k = c0 + col;
                    if (p.mode == PCG_CG) {
                        const double2 told = tT[col];
                        double2 rk = tR[col];
                        rk.x = fma(-alpha_prev, told.x, rk.x);
                        rk.y = fma(-alpha_prev, told.y, rk.y);
                        rr = fma(rk.x, rk.x, fma(rk.y, rk.y, rr));
                        rt = fma(rk.x, t.x, fma(rk.y, t.y, rt));  // Re(conj(r) t)
                        p.r[k] = rk;
                        p.tout[k] = t;
                    } else if (p.mode == PCG_INIT) {
                        p.r[k] = t;
                        p.tout[k] = make_double2(0.0, 0.0);
                    } else {
                        p.tout[k] = t;
                    }
                    qq = fma(t.x, t.x, fma(t.y, t.y, qq));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
    }

    // ---------------------------------------------------------- epilogue
    __syncthreads();  // all stages consumed: the stage ring is free
    double2* sred = reinterpret_cast<double2*>(smem);  // [NG][m]
    double* scal = reinterpret_cast<double*>(smem + size_t(NG) * size_t(m) * 16);
    if (warp < kConsumerWarps) {
#pragma unroll
        for (int e = 0; e < EPL; ++e)
            if (ROW(e) < mi) sred[gq * mi + ROW(e)] = sacc[e];
        if (wig == 0 && lane == 0) {
            scal[gq * 3 + 0] = qq;
            scal[gq * 3 + 1] = rt;
            scal[gq * 3 + 2] = rr;
        }
    }
#undef ROW
    __syncthreads();
    double2* ps = p.part_s + int64_t(blockIdx.x) * m;
    for (int64_t row = threadIdx.x; row < m; row += blockDim.x) {
        double2 acc = sred[row];
        for (int g = 1; g < NG; ++g) acc = c_add(acc, sred[int64_t(g) * m + row]);
        ps[row] = acc;
    }
    if (threadIdx.x == 0) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int g = 0; g < NG; ++g) {
            a0 += scal[g * 3 + 0];
            a1 += scal[g * 3 + 1];
            a2 += scal[g * 3 + 2];
        }
        double* sc = p.part_scal + int64_t(blockIdx.x) * 4;
        sc[0] = a0;
        sc[1] = a1;
        sc[2] = a2;
        sc[3] = 0.0;
    }
}

// ------------------------------------------------------------------ reduce
__global__ void pcg_reduce_kernel(const double2* __restrict__ part_s, const double* __restrict__ part_scal, int parts,
                                  int64_t m, double* __restrict__ red, const CgState* state) {
    if (state && state->done) return;
    const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row < m) {
        double2 acc = part_s[row];
        for (int b = 1; b < parts; ++b) acc = c_add(acc, part_s[int64_t(b) * m + row]);
        reinterpret_cast<double2*>(red)[row] = acc;
    }
    if (blockIdx.x == 0 && threadIdx.x < 4) {
        double acc = 0.0;
        for (int b = 0; b < parts; ++b) acc += part_scal[b * 4 + threadIdx.x];
        red[2 * m + threadIdx.x] = acc;
    }
}

constexpr int kUpdWarps = 8;

__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double2 q = shfl_xor2(v, o);
        v.x += q.x;
        v.y += q.y;
    }
    return v;
}

// upd1 (lsq.cpp:89-98 restated for the fused pass):
//   alpha = gg/qq; u += alpha dir; g -= alpha Rinv^H s; part_gg = ||g||^2 partials.
// init: g = Rinv^H s (s = A c), u = 0, dir_old = 0; rr0 = ||c||^2.
__global__ void __launch_bounds__(kUpdWarps * 32) pcg_upd1_kernel(const double* __restrict__ red,
                                                                 const double2* __restrict__ Rinv, int64_t m,
                                                                 double2* u, double2* g, const double2* dir,
                                                                 double2* dir_old, double* part_gg, CgState* st,
                                                                 double* residual_norms, int init) {
    extern __shared__ double2 s_sh[];
    __shared__ double wsum[kUpdWarps];
    if (st->done) return;
    const double2* s = reinterpret_cast<const double2*>(red);
    const double qq = red[2 * m + 0], rt = red[2 * m + 1], rrk = red[2 * m + 2];
    double alpha = 0.0;
    if (!init) {
        if (qq == 0.0) {  // lsq.cpp:91 -- break before any update
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                st->done = 1;
                st->stop_qq0 = 1;
                st->alpha = 0.0;
                residual_norms[st->iterations] = sqrt(rrk);
                st->rr = rrk;
            }
            return;
        }
        alpha = st->gg / qq;
    }
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s_sh[i] = s[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = int64_t(blockIdx.x) * kUpdWarps + warp;
    double my = 0.0;
    if (j < m) {
        const double2* col = Rinv + j * m;  // column j of Rinv: entries i <= j
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t i = lane; i <= j; i += 32) {
            const double2 a = col[i], b = s_sh[i];
            acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));  // conj(a) * b
            acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
        }
        acc = warp_sum2(acc);
        if (lane == 0) {
            double2 gj;
            if (init) {
                gj = acc;
                u[j] = make_double2(0.0, 0.0);
                dir_old[j] = make_double2(0.0, 0.0);
            } else {
                const double2 dj = dir[j];
                double2 uj = u[j];
                uj.x = fma(alpha, dj.x, uj.x);
                uj.y = fma(alpha, dj.y, uj.y);
                u[j] = uj;
                dir_old[j] = dj;
                gj = g[j];
                gj.x = fma(-alpha, acc.x, gj.x);
                gj.y = fma(-alpha, acc.y, gj.y);
            }
            g[j] = gj;
            my = gj.x * gj.x + gj.y * gj.y;
        }
    }
    if (lane == 0) wsum[warp] = my;
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int w = 0; w < kUpdWarps; ++w) acc += wsum[w];
        part_gg[blockIdx.x] = acc;
        if (blockIdx.x == 0) {
            if (init) {
                st->rr0 = qq;  // INIT pass: qq = ||c||^2
                st->rr = qq;
                st->floor2 = 1e-28 * qq;
                st->iterations = 0;
                st->alpha = 0.0;
                residual_norms[0] = sqrt(qq);
            } else {
                // exact ||r_k||^2 of this pass; estimate of ||r_{k+1}||^2 = ||r_k - alpha t_k||^2
                residual_norms[st->iterations] = sqrt(rrk);
                st->rr = rrk - 2.0 * alpha * rt + alpha * alpha * qq;
                st->alpha = alpha;
                st->iterations += 1;
                st->gg_prev = st->gg;
            }
        }
    }
}

// upd2 (lsq.cpp:99-106): convergence test, beta, dir, and w = Rinv dir for the next pass.
__global__ void __launch_bounds__(kUpdWarps * 32) pcg_upd2_kernel(const double* __restrict__ part_gg, int parts,
                                                                 const double2* __restrict__ Rinv_rows, int64_t m,
                                                                 const double2* g, const double2* dir_old,
                                                                 double2* dir, double2* w, CgState* st, int init) {
    extern __shared__ double2 d_sh[];
    if (st->done) return;
    double ggn = 0.0;
    for (int b = 0; b < parts; ++b) ggn += part_gg[b];  // fixed order, every block
    const double rr = st->rr;
    const double excess = st->dup * ggn;
    const bool conv = excess <= st->tau * fmax(rr - excess, 0.0) || rr <= st->floor2;
    const bool capped = !init && st->iterations >= st->max_iterations;
    if (conv || capped || ggn == 0.0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->done = 1;
            st->converged = conv ? 1 : 0;
            st->excess = excess;
            st->gg = ggn;
        }
        return;
    }
    const double beta = init ? 0.0 : ggn / st->gg_prev;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const double2 gi = g[i], di = dir_old[i];
        d_sh[i] = init ? gi : make_double2(fma(beta, di.x, gi.x), fma(beta, di.y, gi.y));
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = int64_t(blockIdx.x) * kUpdWarps + warp;
    if (i < m) {
        const double2* row = Rinv_rows + i * m;  // row i of Rinv: entries j >= i
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t jj = i + lane; jj < m; jj += 32) {
            const double2 a = row[jj], b = d_sh[jj];
            acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
            acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
        }
        acc = warp_sum2(acc);
        if (lane == 0) {
            w[i] = acc;
            dir[i] = d_sh[i];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->gg = ggn;
        st->excess = excess;
    }
}

// finalize: apply the pending lagged update and take the exact ||r||^2.
__global__ void pcg_finalize_kernel(double2* r, const double2* t, int64_t n, const CgState* st, double* scratch) {
    __shared__ double ws[32];
    const double alpha = st->alpha;
    double acc = 0.0;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        double2 rk = r[k];
        if (alpha != 0.0) {
            const double2 tk = t[k];
            rk.x = fma(-alpha, tk.x, rk.x);
            rk.y = fma(-alpha, tk.y, rk.y);
            r[k] = rk;
        }
        acc = fma(rk.x, rk.x, fma(rk.y, rk.y, acc));
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) s += ws[w];
        scratch[blockIdx.x] = s;
    }
}
__global__ void pcg_finalize_sum_kernel(const double* scratch, int parts, CgState* st) {
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += scratch[b];
    st->rr_final = s;
    st->alpha = 0.0;
}

__global__ void trmv_rows_kernel(const double2* __restrict__ Rr, int64_t m, const double2* __restrict__ u,
                                 double2* __restrict__ y) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = int64_t(blockIdx.x) * kUpdWarps + warp;
    if (i >= m) return;
    const double2* row = Rr + i * m;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t j = i + lane; j < m; j += 32) {
        const double2 a = row[j], b = u[j];
        acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
        acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
    }
    acc = warp_sum2(acc);
    if (lane == 0) y[i] = acc;
}

__global__ void transpose_kernel(const double2* __restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                                 double2* __restrict__ out, int64_t ld_out) {
    __shared__ double2 tile[32][33];
    const int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + threadIdx.x, c = c0 + k;
        if (r < rows && c < cols) tile[k][threadIdx.x] = in[r + c * ld_in];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + threadIdx.x, r = r0 + k;
        if (r < rows && c < cols) out[c + r * ld_out] = tile[threadIdx.x][k];
    }
}

__global__ void init_state_kernel(CgState* st, double tau, double dup, long long max_it) {
    CgState z{};
    z.tau = tau;
    z.dup = dup;
    z.max_iterations = max_it;
    *st = z;
}

template <typename AT, int EPL>
void launch_typed(const PcgPassArgs& a, const PcgPlan& pl, cudaStream_t stream) {
    auto k = pcg_pass_kernel<AT, EPL>;
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem)));
    k<<<pl.grid, kThreads, pl.smem, stream>>>(a, pl.G, pl.cols_per_group, pl.stages, pl.stage_cols);
    MNB_LAUNCH_CHECK();
}

}  // namespace

PcgPlan plan_pcg_pass(int64_t m, int64_t n, int is_real, int num_sms) {
    PcgPlan pl;
    const int esz = is_real ? 8 : 16;
    const int max_epl = is_real ? 8 : 4;
    pl.G = 1;
    while (pl.G < kConsumerWarps && int64_t(32) * pl.G * max_epl < m) pl.G <<= 1;
    int64_t epl = (m + 32 * pl.G - 1) / (32 * pl.G);
    pl.EPL = epl <= 1 ? 1 : epl <= 2 ? 2 : epl <= 4 ? 4 : 8;
    require(int64_t(32) * pl.G * pl.EPL >= m, MNB_ERR_UNSUPPORTED, "pcg pass: m too large for one CTA");
    const int NG = kConsumerWarps / pl.G;
    const int64_t col_bytes = m * esz;
    // stage ~32 KiB, at least one column per group
    int64_t cpg = std::max<int64_t>(1, (32 * 1024) / (NG * col_bytes));
    pl.cols_per_group = int(cpg);
    pl.stage_cols = NG * cpg;
    pl.stages = 6;
    auto fits = [&](int stages) {
        const SmemLayout L = smem_layout(m, pl.stage_cols, esz, stages);
        const size_t epi = size_t(NG) * size_t(m) * 16 + size_t(NG) * 3 * 8;
        return std::max(L.total, epi + 64) <= size_t(220 * 1024);
    };
    while (pl.stages > 2 && !fits(pl.stages)) --pl.stages;
    require(fits(pl.stages), MNB_ERR_UNSUPPORTED, "pcg pass: stage does not fit in shared memory");
    const SmemLayout L = smem_layout(m, pl.stage_cols, esz, pl.stages);
    const size_t epi = size_t(NG) * size_t(m) * 16 + size_t(NG) * 3 * 8;
    pl.smem = std::max(L.total, epi + 64);
    const int64_t max_grid = (n + pl.stage_cols - 1) / pl.stage_cols;
    pl.grid = int(std::max<int64_t>(1, std::min<int64_t>(num_sms, max_grid)));
    return pl;
}

void launch_pcg_pass(const PcgPassArgs& a, const PcgPlan& pl, cudaStream_t stream) {
    if (a.is_real) {
        switch (pl.EPL) {
            case 1: launch_typed<double, 1>(a, pl, stream); break;
            case 2: launch_typed<double, 2>(a, pl, stream); break;
            case 4: launch_typed<double, 4>(a, pl, stream); break;
            default: launch_typed<double, 8>(a, pl, stream); break;
        }
    } else {
        switch (pl.EPL) {
            case 1: launch_typed<double2, 1>(a, pl, stream); break;
            case 2: launch_typed<double2, 2>(a, pl, stream); break;
            case 4: launch_typed<double2, 4>(a, pl, stream); break;
            default: launch_typed<double2, 8>(a, pl, stream); break;
        }
    }
}

void launch_pcg_reduce(const double2* part_s, const double* part_scal, int parts, int64_t m, double* red,
                       const CgState* state, cudaStream_t stream) {
    pcg_reduce_kernel<<<ceil_div(m, 256), 256, 0, stream>>>(part_s, part_scal, parts, m, red, state);
    MNB_LAUNCH_CHECK();
}

int pcg_upd_blocks(int64_t m) { return int(ceil_div(m, kUpdWarps)); }

void launch_pcg_upd1(const double* red, const double2* Rinv, int64_t m, double2* u, double2* g, const double2* dir,
                     double2* dir_old, double* part_gg, CgState* state, double* residual_norms, int init,
                     cudaStream_t stream) {
    const size_t smem = size_t(m) * 16;
    if (smem > 48 * 1024)
        MNB_CUDA(cudaFuncSetAttribute(pcg_upd1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    pcg_upd1_kernel<<<pcg_upd_blocks(m), kUpdWarps * 32, smem, stream>>>(red, Rinv, m, u, g, dir, dir_old, part_gg,
                                                                       state, residual_norms, init);
    MNB_LAUNCH_CHECK();
}

void launch_pcg_upd2(const double* part_gg, int parts_gg, const double2* Rinv_rows, int64_t m, const double2* g,
                     const double2* dir_old, double2* dir, double2* w, CgState* state, int init,
                     cudaStream_t stream) {
    const size_t smem = size_t(m) * 16;
    if (smem > 48 * 1024)
        MNB_CUDA(cudaFuncSetAttribute(pcg_upd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    pcg_upd2_kernel<<<pcg_upd_blocks(m), kUpdWarps * 32, smem, stream>>>(part_gg, parts_gg, Rinv_rows, m, g,
                                                                       dir_old, dir, w, state, init);
    MNB_LAUNCH_CHECK();
}

void launch_pcg_finalize(double2* r, const double2* t, int64_t n, CgState* state, double* scratch,
                         cudaStream_t stream) {
    const int blocks = int(std::min<int64_t>(296, ceil_div(n, 256)));
    pcg_finalize_kernel<<<blocks, 256, 0, stream>>>(r, t, n, state, scratch);
    MNB_LAUNCH_CHECK();
    pcg_finalize_sum_kernel<<<1, 1, 0, stream>>>(scratch, blocks, state);
    MNB_LAUNCH_CHECK();
}

void launch_trmv_rows(const double2* Rinv_rows, int64_t m, const double2* u, double2* y, cudaStream_t stream) {
    trmv_rows_kernel<<<pcg_upd_blocks(m), kUpdWarps * 32, 0, stream>>>(Rinv_rows, m, u, y);
    MNB_LAUNCH_CHECK();
}

void launch_transpose(const double2* in, int64_t rows, int64_t cols, int64_t ld_in, double2* out, int64_t ld_out,
                      cudaStream_t stream) {
    dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, stream>>>(in, rows, cols, ld_in, out, ld_out);
    MNB_LAUNCH_CHECK();
}

void launch_init_state(CgState* st, double tau, double dup, long long max_it, cudaStream_t stream) {
    init_state_kernel<<<1, 1, 0, stream>>>(st, tau, dup, max_it);
    MNB_LAUNCH_CHECK();
}

}  // namespace mnb
