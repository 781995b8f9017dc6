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
constexpr int kThreads = kConsumerWarps * 32;  // no separate producer warp: thread 0 issues the TMA

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

// Columns per batch for a thread owning EPL rows: keeps the two register
// batches (current + next) at <= 16 complex (or 32 real) values per thread.
template <typename AT, int EPL>
__host__ __device__ constexpr int batch_cols() {
    return sizeof(AT) == 16 ? (EPL <= 2 ? 4 : EPL == 4 ? 2 : 1) : (EPL <= 4 ? 4 : 2);
}

struct SmemLayout {
    size_t tileA, tileT, tileR, tileX, stage_bytes, red, bars, total;
};

__host__ __device__ inline SmemLayout smem_layout(int64_t m, int64_t C, int esz, int stages, int V) {
    SmemLayout L;
    const size_t a = size_t(C) * size_t(m) * size_t(esz);
    L.tileA = 0;
    L.tileT = (a + 127) & ~size_t(127);
    L.tileR = L.tileT + ((size_t(C) * 16 + 127) & ~size_t(127));
    L.tileX = L.tileR + ((size_t(C) * 16 + 127) & ~size_t(127));
    L.stage_bytes = L.tileX + ((size_t(C) * 16 + 127) & ~size_t(127));
    L.red = size_t(stages) * L.stage_bytes;  // [groups][2 bufs][G warps][V] doubles = 2 * 16 * V doubles
    L.bars = L.red + size_t(2 * kConsumerWarps * V) * 8;
    L.total = L.bars + size_t(2 * stages) * 8;
    return L;
}

// In-warp transposed reduction of V values (V | 32): afterwards every lane
// holds the warp-wide sum of value index  lane >> (5 - log2 V)  in v[0].
// V-1 + 5-log2(V) shuffles instead of 5 V.
template <int V>
__device__ __forceinline__ void xreduce(double (&v)[V], int lane) {
    int mask = 16;
#pragma unroll
    for (int c = V; c > 1; c >>= 1) {
        const bool up = (lane & mask) != 0;
#pragma unroll
        for (int i = 0; i < c / 2; ++i) {
            const double send = up ? v[i] : v[i + c / 2];
            const double keep = up ? v[i + c / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
        }
        mask >>= 1;
    }
#pragma unroll
    for (; mask > 0; mask >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], mask);
}

template <int V>
__host__ __device__ constexpr int log2c() { return V <= 1 ? 0 : 1 + log2c<V / 2>(); }

// Fused CG pass over this CTA's contiguous column range.
//
// A group of G consumer warps owns all m rows (thread: EPL rows, stride
// 32 G); NG = 16/G groups split each shared-memory stage, K columns each.
// Per batch of K columns a warp forms K partial dot products, reduces them
// in-warp (xreduce), publishes them to shared memory, and -- one named
// barrier later -- sums the G warp partials into t, then does the axpy.
// A stage is handed back to the TMA producer (thread 0) as soon as it sits
// in registers.  All sums run in a fixed order (bitwise reproducible).
//
// GT != 0: compile-time group width with m == 32*GT*EPL exactly (every
// BASELINE shape), so shared-memory offsets are immediates and no row is
// masked; GT == 0 is the generic kernel (runtime G, masked rows).
template <typename AT, int EPL, int GT>
__global__ void __launch_bounds__(kThreads, 1) pcg_pass_kernel(const PcgPassArgs p, int g_rt, int stages, int64_t C_rt,
                                                               int64_t per) {
    constexpr int K = batch_cols<AT, EPL>();
    constexpr int V = 2 * K;
    // exact shapes: one batch per group per stage (plan_pcg_pass), so the stage
    // geometry folds to immediates
    const int64_t C = GT ? int64_t(kConsumerWarps / (GT ? GT : 1)) * K : C_rt;
    extern __shared__ __align__(128) unsigned char smem[];
    if (p.state && p.state->done) return;  // uniform: converged loops cost one launch
    const int G = GT ? GT : g_rt;
    const int mi = GT ? 32 * GT * EPL : int(p.m);
    const int64_t m = mi;
    constexpr int esz = int(sizeof(AT));
    const SmemLayout L = smem_layout(m, C, esz, stages, V);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + stages;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NG = kConsumerWarps / G;
    const int64_t cb = min(p.n, int64_t(blockIdx.x) * per), ce = min(p.n, cb + per);
    const int64_t nstage = (ce - cb + C - 1) / C;
    const int mode = p.mode;
    const bool init = mode == PCG_INIT;
    const bool need_t = init || mode == PCG_CG;
    const bool need_r = mode == PCG_CG;
    const bool need_x = mode == PCG_CG && p.x != nullptr;  // x = sum_k alpha_k t_k, updated lagged like r
    const double alpha_prev = (mode == PCG_CG && p.state) ? p.state->alpha : 0.0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // Producer (thread 0): fill stage s into `slot`.  The first `stages`
    // fills are issued here; later ones from the consumer loop, each after
    // every warp has moved the slot's previous occupant into registers.
    auto produce = [&](int64_t s, int slot) {
        const int64_t c0 = cb + s * C;
        const int64_t cc = min(C, ce - c0);
        unsigned char* st = smem + slot * L.stage_bytes;
        const size_t abytes = size_t(cc) * size_t(m) * esz;
        const uint32_t abulk = uint32_t(abytes & ~size_t(15));
        const unsigned char* src = static_cast<const unsigned char*>(p.A) + size_t(c0) * size_t(m) * esz;
        if (abytes != abulk)  // odd real tail: 8 bytes by hand, published by the arrive below
            *reinterpret_cast<double*>(st + L.tileA + abulk) = __ldg(reinterpret_cast<const double*>(src + abulk));
        const uint32_t vbytes = uint32_t(cc * 16);
        mbar_expect_tx(&full[slot], abulk + (need_t ? vbytes : 0u) + (need_r ? vbytes : 0u) + (need_x ? vbytes : 0u));
        if (abulk) bulk_g2s(st + L.tileA, src, abulk, &full[slot]);
        if (need_t) bulk_g2s(st + L.tileT, p.tin + c0, vbytes, &full[slot]);
        if (need_r) bulk_g2s(st + L.tileR, p.r + c0, vbytes, &full[slot]);
        if (need_x) bulk_g2s(st + L.tileX, p.x + c0, vbytes, &full[slot]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < nstage && s < stages; ++s) produce(s, s);

    // ---------------------------------------------------------- consumers
    const int gq = warp / G, wig = warp % G;
    const int row0 = wig * 32 + lane, rstep = 32 * G;
    double2 wreg[EPL], sacc[EPL];
    // Real A at exact shapes: a lane owns EPL/2 PAIRS of adjacent rows, so the
    // stage is read with 16-byte shared loads (half the load instructions).
    constexpr bool PAIR = sizeof(AT) == 8 && GT != 0 && EPL % 2 == 0;
#define ROW(e) (PAIR ? 2 * (row0 + ((e) >> 1) * rstep) + ((e) & 1) : row0 + (e) * rstep)
#define ROW_OK(e) (GT != 0 || ROW(e) < mi)
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        sacc[e] = make_double2(0.0, 0.0);
        wreg[e] = make_double2(0.0, 0.0);
    }
    double qq = 0.0, rt = 0.0, rr = 0.0;  // per-lane partials (lanes < K of warp wig == 0)
    double* red = reinterpret_cast<double*>(smem + L.red) + size_t(gq) * 2 * G * V;  // [2][G][V]
    if (nstage > 0) {
        if (!init) {
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (ROW_OK(e)) wreg[e] = p.w[ROW(e)];
        }
        AT a[K][EPL];
        double v[V];
        int lslot = 0, pslot = 0, cslot = 0;  // consumer load slot, producer refill slot, current batch slot
        uint32_t lph = 0, pph = 0;
        int64_t c0 = cb;

        // The slot of batch s is released when batch s+1 is loaded, so the
        // epilogue of batch s can still read its t_old / r / c from the stage.
        // a[][] <- the batch's columns from stage st (cc columns in the stage)
        auto fetch = [&](const unsigned char* st, int64_t cc) {
            const AT* tA = reinterpret_cast<const AT*>(st + L.tileA) + gq * K * mi + (PAIR ? 2 * row0 : row0);
            if constexpr (PAIR) {
                const int have = cc == C ? K : int(cc) - gq * K;
                if (cc == C) {
#pragma unroll
                    for (int k = 0; k < K; ++k)
#pragma unroll
                        for (int e = 0; e < EPL; e += 2) {
                            const double2 pr = *reinterpret_cast<const double2*>(
                                reinterpret_cast<const double*>(tA) + k * mi + e * rstep);
                            reinterpret_cast<double*>(&a[k][e])[0] = pr.x;
                            reinterpret_cast<double*>(&a[k][e + 1])[0] = pr.y;
                        }
                    return;
                }
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int e = 0; e < EPL; e += 2) {
                        const double2 pr = k < have ? *reinterpret_cast<const double2*>(
                                                          reinterpret_cast<const double*>(tA) + k * mi + e * rstep)
                                                    : make_double2(0.0, 0.0);
                        reinterpret_cast<double*>(&a[k][e])[0] = pr.x;
                        reinterpret_cast<double*>(&a[k][e + 1])[0] = pr.y;
                    }
            } else if (cc == C) {  // uniform: every stage but possibly the last
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int e = 0; e < EPL; ++e) a[k][e] = ROW_OK(e) ? tA[k * mi + e * rstep] : zero_of<AT>();
            } else {
                const int have = int(cc) - gq * K;  // columns of this group present in the stage
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int e = 0; e < EPL; ++e)
                        a[k][e] = (k < have && ROW_OK(e)) ? tA[k * mi + e * rstep] : zero_of<AT>();
            }
        };
        // The slot of batch s is released when batch s+1 is loaded, so the
        // epilogue of batch s can still read its t_old / r / c from the stage.
        auto load = [&](int64_t cc, bool release_prev) {
            if (release_prev) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[cslot]);
            }
            mbar_wait(&full[lslot], lph);
            fetch(smem + lslot * L.stage_bytes, cc);
            cslot = lslot;
            if (++lslot == stages) {
                lslot = 0;
                lph ^= 1u;
            }
        };
        // partial dot products of the batch, reduced in-warp and published
        auto dots = [&](int buf) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double2 part = make_double2(0.0, 0.0);
#pragma unroll
                for (int e = 0; e < EPL; ++e) dot_acc<AT>(part, a[k][e], wreg[e]);
                v[2 * k] = part.x;
                v[2 * k + 1] = part.y;
            }
            xreduce<V>(v, lane);
            if (G > 1 && (lane & ((32 / V) - 1)) == 0) red[(buf * G + wig) * V + (lane >> (5 - log2c<V>()))] = v[0];
        };
        // t of the batch from the published partials (or from v when G == 1)
        auto gather_t = [&](int buf, double2 (&t)[K]) {
            double acc;
            if (G > 1) {
                // G*V partials: lane L sums entries L, L+32, ... (all of value L % V)
                const double* rb = red + buf * G * V;
                acc = rb[lane < G * V ? lane : 0];
                if (lane >= G * V) acc = 0.0;
#pragma unroll
                for (int j = 1; j < (16 * V) / 32; ++j)
                    if (lane + 32 * j < G * V) acc += rb[lane + 32 * j];
#pragma unroll
                for (int mask = V; mask < 32; mask <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, mask);
#pragma unroll
                for (int k = 0; k < K; ++k)
                    t[k] = make_double2(__shfl_sync(0xffffffffu, acc, 2 * k), __shfl_sync(0xffffffffu, acc, 2 * k + 1));
            } else {
                acc = v[0];
                constexpr int sh = 5 - log2c<V>();
#pragma unroll
                for (int k = 0; k < K; ++k)
                    t[k] = make_double2(__shfl_sync(0xffffffffu, acc, (2 * k) << sh),
                                        __shfl_sync(0xffffffffu, acc, (2 * k + 1) << sh));
            }
        };

        int64_t cc = min(C, ce - c0);
        load(cc, false);
        if (!init) dots(0);
        for (int64_t s = 0; s < nstage; ++s) {
            const int buf = int(s & 1);
            if (G > 1 && !init) named_bar(1 + gq, G * 32);
            const unsigned char* cst = smem + cslot * L.stage_bytes;
            const double2* tT = reinterpret_cast<const double2*>(cst + L.tileT) + gq * K;
            const double2* tR = reinterpret_cast<const double2*>(cst + L.tileR) + gq * K;
            const double2* tX = reinterpret_cast<const double2*>(cst + L.tileX) + gq * K;
            double2 t[K];
            if (init) {
                const int have = int(cc) - gq * K;
#pragma unroll
                for (int k = 0; k < K; ++k) t[k] = k < have ? tT[k] : make_double2(0.0, 0.0);
            } else {
                gather_t(buf, t);
            }
#ifdef MNB_PCG_REREAD
            // the batch is still in its stage: read it again rather than hold it across the barrier
            if (!init) fetch(cst, cc);
#endif
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int e = 0; e < EPL; ++e) axpy_acc<AT>(sacc[e], a[k][e], t[k]);
            // per-column epilogue (lane k < K of the group's first warp owns column k)
            if (wig == 0 && lane < K && gq * K + lane < cc) {
                double2 tk = t[0];
#pragma unroll
                for (int k = 1; k < K; ++k)
                    if (lane == k) tk = t[k];
                const int64_t col = c0 + gq * K + lane;
                if (mode == PCG_CG) {
                    const double2 told = tT[lane];
                    double2 rk = tR[lane];
                    rk.x = fma(-alpha_prev, told.x, rk.x);
                    rk.y = fma(-alpha_prev, told.y, rk.y);
                    rr = fma(rk.x, rk.x, fma(rk.y, rk.y, rr));
                    rt = fma(rk.x, tk.x, fma(rk.y, tk.y, rt));  // Re(conj(r) t)
                    p.r[col] = rk;
                    p.tout[col] = tk;
                    if (need_x) {
                        double2 xk = tX[lane];
                        xk.x = fma(alpha_prev, told.x, xk.x);
                        xk.y = fma(alpha_prev, told.y, xk.y);
                        p.x[col] = xk;
                    }
                } else if (init) {
                    p.r[col] = tk;
                    p.tout[col] = make_double2(0.0, 0.0);
                    if (p.x) p.x[col] = make_double2(0.0, 0.0);
                } else {
                    p.tout[col] = tk;
                }
                qq = fma(tk.x, tk.x, fma(tk.y, tk.y, qq));
            }
            if (s + 1 < nstage) {
                c0 += C;
                cc = min(C, ce - c0);
                load(cc, true);
                if (threadIdx.x == 0 && s + stages < nstage) {
                    mbar_wait(&empty[pslot], pph);
                    produce(s + stages, pslot);
                    if (++pslot == stages) {
                        pslot = 0;
                        pph ^= 1u;
                    }
                }
                if (!init) dots(buf ^ 1);
            }
        }
    }

    // ---------------------------------------------------------- epilogue
    __syncthreads();  // all stages consumed: the stage ring is free
    double2* sred = reinterpret_cast<double2*>(smem);  // [NG][m]
    double* scal = reinterpret_cast<double*>(smem + size_t(NG) * size_t(m) * 16);
#pragma unroll
    for (int e = 0; e < EPL; ++e)
        if (ROW_OK(e)) sred[gq * mi + ROW(e)] = sacc[e];
    if (wig == 0) {
        // lanes >= K hold zeros; fixed-order butterfly
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            qq += __shfl_xor_sync(0xffffffffu, qq, o);
            rt += __shfl_xor_sync(0xffffffffu, rt, o);
            rr += __shfl_xor_sync(0xffffffffu, rr, o);
        }
        if (lane == 0) {
            scal[gq * 3 + 0] = qq;
            scal[gq * 3 + 1] = rt;
            scal[gq * 3 + 2] = rr;
        }
    }
#undef ROW_OK
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
// s = sum of the per-CTA partials.  32 rows x 8 part slices per block (each thread sums
// every 8th part, then the 8 slices in order): ~19 independent loads per thread instead of
// a 148-long dependent chain on 8 blocks.  Fixed order: deterministic.
constexpr int kRedRows = 32, kRedSlices = 8;
__global__ void __launch_bounds__(kRedRows * kRedSlices) pcg_reduce_kernel(const double2* __restrict__ part_s,
                                                                         const double* __restrict__ part_scal,
                                                                         int parts, int64_t m, double* __restrict__ red,
                                                                         const CgState* state) {
    if (state && state->done) return;
    __shared__ double2 sh[kRedSlices][kRedRows];
    const int rr = int(threadIdx.x) % kRedRows, sl = int(threadIdx.x) / kRedRows;
    const int64_t row = int64_t(blockIdx.x) * kRedRows + rr;
    double2 acc = make_double2(0.0, 0.0);
    if (row < m)
        for (int b = sl; b < parts; b += kRedSlices) acc = c_add(acc, part_s[int64_t(b) * m + row]);
    sh[sl][rr] = acc;
    __syncthreads();
    if (sl == 0 && row < m) {
        double2 t = sh[0][rr];
#pragma unroll
        for (int k = 1; k < kRedSlices; ++k) t = c_add(t, sh[k][rr]);
        reinterpret_cast<double2*>(red)[row] = t;
    }
    if (blockIdx.x == 0 && threadIdx.x < 4) {
        double a = 0.0;
        for (int b = 0; b < parts; ++b) a += part_scal[b * 4 + threadIdx.x];
        red[2 * m + threadIdx.x] = a;
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
                                                                 double* residual_norms, int init, double2* ax) {
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
        // four independent accumulators (four loads in flight per lane), combined in fixed order
        double2 ac[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                         make_double2(0.0, 0.0)};
        int64_t i = lane;
        for (; i + 96 <= j; i += 128) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double2 a = col[i + 32 * k], b = s_sh[i + 32 * k];
                ac[k].x = fma(a.x, b.x, fma(a.y, b.y, ac[k].x));  // conj(a) * b
                ac[k].y = fma(a.x, b.y, fma(-a.y, b.x, ac[k].y));
            }
        }
        for (; i <= j; i += 32) {
            const double2 a = col[i], b = s_sh[i];
            ac[0].x = fma(a.x, b.x, fma(a.y, b.y, ac[0].x));
            ac[0].y = fma(a.x, b.y, fma(-a.y, b.x, ac[0].y));
        }
        double2 acc = c_add(c_add(ac[0], ac[1]), c_add(ac[2], ac[3]));
        acc = warp_sum2(acc);
        if (lane == 0) {
            double2 gj;
            if (init) {
                gj = acc;
                u[j] = make_double2(0.0, 0.0);
                dir_old[j] = make_double2(0.0, 0.0);
                if (ax) ax[j] = make_double2(0.0, 0.0);
            } else {
                if (ax) {  // A x = sum_k alpha_k s_k (the Step-5 product, src/solver.cpp:122)
                    double2 axj = ax[j];
                    axj.x = fma(alpha, s_sh[j].x, axj.x);
                    axj.y = fma(alpha, s_sh[j].y, axj.y);
                    ax[j] = axj;
                }
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
        double2 ac[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                         make_double2(0.0, 0.0)};
        int64_t jj = i + lane;
        for (; jj + 96 < m; jj += 128) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double2 a = row[jj + 32 * k], b = d_sh[jj + 32 * k];
                ac[k].x = fma(a.x, b.x, fma(-a.y, b.y, ac[k].x));
                ac[k].y = fma(a.x, b.y, fma(a.y, b.x, ac[k].y));
            }
        }
        for (; jj < m; jj += 32) {
            const double2 a = row[jj], b = d_sh[jj];
            ac[0].x = fma(a.x, b.x, fma(-a.y, b.y, ac[0].x));
            ac[0].y = fma(a.x, b.y, fma(a.y, b.x, ac[0].y));
        }
        double2 acc = c_add(c_add(ac[0], ac[1]), c_add(ac[2], ac[3]));
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
__global__ void pcg_finalize_kernel(double2* r, const double2* t, double2* x, int64_t n, const CgState* st,
                                    double* scratch) {
    __shared__ double ws[32], wx[32];
    const double alpha = st->alpha;
    double acc = 0.0, accx = 0.0;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        double2 rk = r[k];
        const double2 tk = alpha != 0.0 ? t[k] : make_double2(0.0, 0.0);
        if (alpha != 0.0) {
            rk.x = fma(-alpha, tk.x, rk.x);
            rk.y = fma(-alpha, tk.y, rk.y);
            r[k] = rk;
        }
        acc = fma(rk.x, rk.x, fma(rk.y, rk.y, acc));
        if (x) {
            double2 xk = x[k];
            if (alpha != 0.0) {
                xk.x = fma(alpha, tk.x, xk.x);
                xk.y = fma(alpha, tk.y, xk.y);
                x[k] = xk;
            }
            accx = fma(xk.x, xk.x, fma(xk.y, xk.y, accx));
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        accx += __shfl_xor_sync(0xffffffffu, accx, o);
    }
    if ((threadIdx.x & 31) == 0) {
        ws[threadIdx.x >> 5] = acc;
        wx[threadIdx.x >> 5] = accx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0, sx = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            s += ws[w];
            sx += wx[w];
        }
        scratch[2 * blockIdx.x] = s;
        scratch[2 * blockIdx.x + 1] = sx;
    }
}
__global__ void pcg_finalize_sum_kernel(const double* scratch, int parts, CgState* st) {
    double s = 0.0, sx = 0.0;
    for (int b = 0; b < parts; ++b) {
        s += scratch[2 * b];
        sx += scratch[2 * b + 1];
    }
    st->rr_final = s;
    st->xx_final = sx;
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

template <typename AT, int EPL, int GT>
void launch_typed(const PcgPassArgs& a, const PcgPlan& pl, cudaStream_t stream) {
    auto k = pcg_pass_kernel<AT, EPL, GT>;
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem)));
    k<<<pl.grid, kThreads, pl.smem, stream>>>(a, pl.G, pl.stages, pl.stage_cols, pl.per_cta);
    MNB_LAUNCH_CHECK();
}

// Exact shapes m == 32*G*EPL get the compile-time-G kernel; the rest the generic one.
template <typename AT, int EPL>
void launch_epl(const PcgPassArgs& a, const PcgPlan& pl, cudaStream_t stream) {
    const bool exact = a.m == int64_t(32) * pl.G * EPL;
    if (exact) {
        if constexpr (EPL == 4 || EPL == 8) {
            switch (pl.G) {
                case 2: return launch_typed<AT, EPL, 2>(a, pl, stream);
                case 4: return launch_typed<AT, EPL, 4>(a, pl, stream);
                case 8: return launch_typed<AT, EPL, 8>(a, pl, stream);
                case 16: return launch_typed<AT, EPL, 16>(a, pl, stream);
                default: break;
            }
        }
        if (pl.G == 1) return launch_typed<AT, EPL, 1>(a, pl, stream);
    }
    launch_typed<AT, EPL, 0>(a, pl, stream);
}

}  // namespace

PcgPlan plan_pcg_pass(int64_t m, int64_t n, int is_real, int num_sms) {
    PcgPlan pl;
    const int esz = is_real ? 8 : 16;
    // rows per thread: up to 4 (complex) / 8 (real) before the group widens to 16 warps
    const int pref_epl = is_real ? 8 : 4;
    pl.G = 1;
    while (pl.G < kConsumerWarps && int64_t(32) * pl.G * pref_epl < m) pl.G <<= 1;
    int64_t epl = (m + 32 * pl.G - 1) / (32 * pl.G);
    pl.EPL = epl <= 1 ? 1 : epl <= 2 ? 2 : epl <= 4 ? 4 : 8;
    require(int64_t(32) * pl.G * pl.EPL >= m, MNB_ERR_UNSUPPORTED,
            "pcg pass: m = " + std::to_string(m) + " exceeds one CTA's rows (max " +
                std::to_string(32 * kConsumerWarps * 8) + ")");
    const int K = is_real ? (pl.EPL == 1 ? batch_cols<double, 1>() : pl.EPL == 2 ? batch_cols<double, 2>()
                             : pl.EPL == 4 ? batch_cols<double, 4>() : batch_cols<double, 8>())
                          : (pl.EPL == 1 ? batch_cols<double2, 1>() : pl.EPL == 2 ? batch_cols<double2, 2>()
                             : pl.EPL == 4 ? batch_cols<double2, 4>() : batch_cols<double2, 8>());
    const int NG = kConsumerWarps / pl.G;
    pl.K = K;
    pl.stage_cols = int64_t(NG) * K;  // one batch per group per stage
    const int64_t col_bytes = m * esz;
    auto fits = [&](int stages) {
        const SmemLayout L = smem_layout(m, pl.stage_cols, esz, stages, 2 * K);
        const size_t epi = size_t(NG) * size_t(m) * 16 + size_t(NG) * 3 * 8;
        return std::max(L.total, epi + 64) <= size_t(220 * 1024);
    };
    // ~192 KiB of stages in flight per SM (the ring is released as soon as a stage is in registers)
    pl.stages = int(std::max<int64_t>(2, std::min<int64_t>(8, (192 * 1024) / std::max<int64_t>(1, pl.stage_cols * col_bytes))));
    while (pl.stages > 2 && !fits(pl.stages)) --pl.stages;
    require(fits(pl.stages), MNB_ERR_UNSUPPORTED, "pcg pass: stage does not fit in shared memory");
    const SmemLayout L = smem_layout(m, pl.stage_cols, esz, pl.stages, 2 * K);
    const size_t epi = size_t(NG) * size_t(m) * 16 + size_t(NG) * 3 * 8;
    pl.smem = std::max(L.total, epi + 64);
    const int64_t max_grid = (n + pl.stage_cols - 1) / pl.stage_cols;
    pl.grid = int(std::max<int64_t>(1, std::min<int64_t>(num_sms, max_grid)));
    // contiguous columns per CTA; even so that a real A with odd m stays 16-byte aligned for TMA
    pl.per_cta = (n + pl.grid - 1) / pl.grid;
    pl.per_cta += pl.per_cta & 1;
    pl.grid = int(std::max<int64_t>(1, (n + pl.per_cta - 1) / pl.per_cta));
    return pl;
}

void launch_pcg_pass(const PcgPassArgs& a, const PcgPlan& pl, cudaStream_t stream) {
    if (a.is_real) {
        switch (pl.EPL) {
            case 1: launch_epl<double, 1>(a, pl, stream); break;
            case 2: launch_epl<double, 2>(a, pl, stream); break;
            case 4: launch_epl<double, 4>(a, pl, stream); break;
            default: launch_epl<double, 8>(a, pl, stream); break;
        }
    } else {
        switch (pl.EPL) {
            case 1: launch_epl<double2, 1>(a, pl, stream); break;
            case 2: launch_epl<double2, 2>(a, pl, stream); break;
            case 4: launch_epl<double2, 4>(a, pl, stream); break;
            default: launch_epl<double2, 8>(a, pl, stream); break;
        }
    }
}

void launch_pcg_reduce(const double2* part_s, const double* part_scal, int parts, int64_t m, double* red,
                       const CgState* state, cudaStream_t stream) {
    pcg_reduce_kernel<<<ceil_div(m, kRedRows), kRedRows * kRedSlices, 0, stream>>>(part_s, part_scal, parts, m, red,
                                                                                   state);
    MNB_LAUNCH_CHECK();
}

int pcg_upd_blocks(int64_t m) { return int(ceil_div(m, kUpdWarps)); }

void launch_pcg_upd1(const double* red, const double2* Rinv, int64_t m, double2* u, double2* g, const double2* dir,
                     double2* dir_old, double* part_gg, CgState* state, double* residual_norms, int init,
                     cudaStream_t stream, double2* ax) {
    const size_t smem = size_t(m) * 16;
    if (smem > 48 * 1024)
        MNB_CUDA(cudaFuncSetAttribute(pcg_upd1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    pcg_upd1_kernel<<<pcg_upd_blocks(m), kUpdWarps * 32, smem, stream>>>(red, Rinv, m, u, g, dir, dir_old, part_gg,
                                                                       state, residual_norms, init, ax);
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

void launch_pcg_finalize(double2* r, const double2* t, double2* x, int64_t n, CgState* state, double* scratch,
                         cudaStream_t stream) {
    const int blocks = int(std::min<int64_t>(296, ceil_div(n, 256)));
    pcg_finalize_kernel<<<blocks, 256, 0, stream>>>(r, t, x, n, state, scratch);
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
