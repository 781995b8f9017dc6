// Sketch-QR kernels (cholqr.cuh): blocked upper Cholesky, triangular inverse and the
// device-resident refinement loops, each ONE persistent cooperative launch whose phases are
// separated by grid barriers.  The m x m factors are L2-resident at every BASELINE shape
// (1 MiB at c2 ... 256 MiB at c5 only exceeds it), so the phases stream them from L2; the host
// reads one status record per sketch instead of steering a chain of library calls.
//
//   chol_upper_kernel   right-looking, 32-wide block rows.  Per block row: every CTA factors the
//                       32 x 32 diagonal block redundantly in shared memory (identical
//                       arithmetic, so no barrier is needed to publish it), a warp per column
//                       solves the row panel by forward substitution with lane shuffles, then
//                       64 x 64 tiles of the trailing Hermitian update are spread over the grid.
//   trtri_upper_kernel  X = R^{-1} bottom-up: 32 x 32 diagonal inverses (a warp per column),
//                       then log2(m / 32) doubling levels X12 = -X11 (R12 X22), each two
//                       grid-wide tile products that skip the zero halves of the triangles.
//   sketch_refine_kernel  Step 2's corrected seminormal equations (src/solver.cpp:93-96) or the
//                       one-pass preconditioner's check ||Q1^H Q1 - I|| (src/lsq.cpp:58-69) as
//                       four GEMV phases per step over the sketch and R1^{-1}; stop decisions
//                       are replicated in every CTA from fixed-order sums (bitwise reproducible).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "cholqr.cuh"

namespace mnb {

namespace {

namespace cg = cooperative_groups;

constexpr int NB = 32;        // Cholesky / inverse block
constexpr int LDD = NB + 1;   // padded row of the diagonal block in shared memory
constexpr int TB = 64;        // tile of the grid-wide products
constexpr int KC = 32;        // k chunk of a tile product
constexpr int LDT = TB + 1;   // padded tile row in shared memory
constexpr int TH = 256;
constexpr int NW = TH / 32;
constexpr double kU = 2.220446049250313e-16;

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {  // acc += a b
    acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ void cmac_conj(double2& acc, double2 a, double2 b) {  // acc += conj(a) b
    acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
}
__device__ __forceinline__ double2 crecip(double2 d) {
    const double s = 1.0 / (d.x * d.x + d.y * d.y);
    return make_double2(d.x * s, -d.y * s);
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}
__device__ __forceinline__ double warp_sum1(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum in a fixed order (warp butterflies, then the NW warp sums in order); every
// thread gets the result.  red: NW doubles of shared memory.
__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum1(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) s += red[q];
    return s;
}

// acc[a][b] += sum_{k in [k_lo, k_hi)} opA(i, k) B(k, j) for the 64 x 64 tile entries
// i = tr + 16 a, j = tc + 16 b of this thread.  opA(i, k) = conj(A[k + i lda]) (TRANS) or
// A[i + k lda]; B(k, j) = B[k + j ldb].  Entries beyond rows_valid / cols_valid read as zero.
// Operands may have been written by other CTAs earlier in the same launch: L2 loads only.
template <bool TRANS>
__device__ __forceinline__ void tile_mm(const double2* A, int64_t lda, const double2* B, int64_t ldb, int k_lo,
                                        int k_hi, int rows_valid, int cols_valid, double2* As, double2* Bs,
                                        double2 (&acc)[4][4]) {
    const int t = threadIdx.x, tr = t & 15, tc = t >> 4;
    for (int kc = k_lo; kc < k_hi; kc += KC) {
        __syncthreads();
        if (TRANS) {
            const int k = t & 31;
            for (int i = t >> 5; i < TB; i += TH / 32) {
                double2 v = make_double2(0.0, 0.0);
                if (kc + k < k_hi && i < rows_valid) {
                    v = __ldcg(A + (kc + k) + int64_t(i) * lda);
                    v.y = -v.y;
                }
                As[k * LDT + i] = v;
            }
        } else {
            const int i = t & 63;
            for (int k = t >> 6; k < KC; k += TH / 64) {
                double2 v = make_double2(0.0, 0.0);
                if (kc + k < k_hi && i < rows_valid) v = __ldcg(A + i + int64_t(kc + k) * lda);
                As[k * LDT + i] = v;
            }
        }
        {
            const int k = t & 31;
            for (int j = t >> 5; j < TB; j += TH / 32) {
                double2 v = make_double2(0.0, 0.0);
                if (kc + k < k_hi && j < cols_valid) v = __ldcg(B + (kc + k) + int64_t(j) * ldb);
                Bs[k * LDT + j] = v;
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < KC; ++k) {
            double2 a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = As[k * LDT + tr + 16 * q];
                b[q] = Bs[k * LDT + tc + 16 * q];
            }
#pragma unroll
            for (int qa = 0; qa < 4; ++qa)
#pragma unroll
                for (int qb = 0; qb < 4; ++qb) cmac(acc[qa][qb], a[qa], b[qb]);
        }
    }
}

__device__ __forceinline__ void zero_acc(double2 (&acc)[4][4]) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------- Cholesky
__global__ void __launch_bounds__(TH, 1)
chol_upper_kernel(double2* G, int64_t m, int64_t ld, double shift_factor, double rank_rows, CholStatus* st) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double2 smem[];
    double2* W = smem;              // [NB][LDD] the diagonal block while it is eliminated
    double2* As = W + NB * LDD;     // [KC][LDT]
    double2* Bs = As + KC * LDT;    // [KC][LDT]
    double2* D = Bs + KC * LDT;     // [NB][LDD] its factor R_kk
    __shared__ double red[NW];
    __shared__ double rdiag[NB];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int ng = gridDim.x, c = blockIdx.x;

    double acc = 0.0;
    for (int64_t j = t; j < m; j += TH) acc += __ldcg(G + j + j * ld).x;
    const double tr = block_sum(acc, red);
    const double shift = shift_factor != 0.0 ? shift_factor * tr : 0.0;
    double dmin = 1e300, dmax = 0.0;  // thread 0's copy is reported
    int info = 0;

    for (int64_t k0 = 0; k0 < m; k0 += NB) {
        const int nb = int(imin64(NB, m - k0));
        // (A) the diagonal block: load its upper triangle (+ shift), factor it in shared memory
        __syncthreads();
        for (int e = t; e < NB * NB; e += TH) {
            const int i = e % NB, j = e / NB;
            double2 v = make_double2(0.0, 0.0);
            if (i <= j && j < nb) {
                v = __ldcg(G + (k0 + i) + (k0 + j) * ld);
                if (i == j) v = make_double2(v.x + shift, 0.0);
            }
            W[i * LDD + j] = v;
            D[i * LDD + j] = make_double2(0.0, 0.0);
        }
        // one barrier per pivot: row j of W is final when step j starts and is only read in it
        // (the scaled row goes to D, the rows below take the rank-1 update with 1 / pivot)
        for (int j = 0; j < nb; ++j) {
            __syncthreads();
            const double piv = W[j * LDD + j].x;
            if (!(piv > 0.0) || !(piv < 1e300)) {  // not positive definite (or not finite): potrf's info
                info = int(k0) + j + 1;
                break;
            }
            const double rinv = rsqrt(piv), r = piv * rinv, pinv = rinv * rinv;
            if (t == 0) rdiag[j] = rinv;
            const int cc = t % NB;
            for (int i = t / NB; i < nb; i += TH / NB) {
                if (i == j) {
                    if (cc > j && cc < nb) {
                        const double2 v = W[j * LDD + cc];
                        D[j * LDD + cc] = make_double2(v.x * rinv, v.y * rinv);
                    } else if (cc == j) {
                        D[j * LDD + j] = make_double2(r, 0.0);
                    }
                } else if (i > j && cc >= i && cc < nb) {
                    const double2 a = W[j * LDD + i], b = W[j * LDD + cc];
                    double2 d = W[i * LDD + cc];
                    d.x = fma(-pinv, fma(a.x, b.x, a.y * b.y), d.x);   // conj(a) b / pivot
                    d.y = fma(-pinv, fma(a.x, b.y, -a.y * b.x), d.y);
                    W[i * LDD + cc] = d;
                }
            }
            dmin = fmin(dmin, r);
            dmax = fmax(dmax, r);
        }
        if (info) break;  // every CTA factored the same block the same way: uniform over the grid
        __syncthreads();
        if (c == 0) {
            for (int e = t; e < NB * NB; e += TH) {
                const int i = e % NB, j = e / NB;
                if (i < nb && j < nb) G[(k0 + i) + (k0 + j) * ld] = i <= j ? D[i * LDD + j] : make_double2(0.0, 0.0);
            }
        }
        // (B) the row panel R[k, c] = R_kk^{-H} G[k, c]: a warp per column, forward substitution
        const int64_t k1 = k0 + nb;
        for (int64_t col = k1 + int64_t(warp) * ng + c; col < m; col += int64_t(NW) * ng) {
            double2 y = lane < nb ? __ldcg(G + (k0 + lane) + col * ld) : make_double2(0.0, 0.0);
            for (int k = 0; k < nb; ++k) {
                if (lane == k) {
                    y.x *= rdiag[k];
                    y.y *= rdiag[k];
                }
                const double2 yk = shfl2(y, k);
                if (lane > k && lane < nb) {
                    const double2 a = D[k * LDD + lane];
                    y.x -= fma(a.x, yk.x, a.y * yk.y);   // conj(R[k, lane]) y_k
                    y.y -= fma(a.x, yk.y, -a.y * yk.x);
                }
            }
            if (lane < nb) G[(k0 + lane) + col * ld] = y;
        }
        grid.sync();
        // (C) trailing update G[i, j] -= R[k, i]^H R[k, j] over 64 x 64 tiles of the upper triangle
        const int64_t rem = m - k1;
        if (rem > 0) {
            const int nt = int((rem + TB - 1) / TB);
            const int tiles = nt * (nt + 1) / 2;
            for (int tile = c; tile < tiles; tile += ng) {
                int J = 0;
                while ((J + 1) * (J + 2) / 2 <= tile) ++J;
                const int I = tile - J * (J + 1) / 2;
                const int64_t r0 = k1 + int64_t(I) * TB, c0 = k1 + int64_t(J) * TB;
                double2 a4[4][4];
                zero_acc(a4);
                tile_mm<true>(G + k0 + r0 * ld, ld, G + k0 + c0 * ld, ld, 0, nb, int(imin64(TB, m - r0)),
                              int(imin64(TB, m - c0)), As, Bs, a4);
                const int tr_ = t & 15, tc_ = t >> 4;
#pragma unroll
                for (int qa = 0; qa < 4; ++qa)
#pragma unroll
                    for (int qb = 0; qb < 4; ++qb) {
                        const int64_t row = r0 + tr_ + 16 * qa, col = c0 + tc_ + 16 * qb;
                        if (row < m && col < m && row <= col) {
                            double2 g = __ldcg(G + row + col * ld);
                            g.x -= a4[qa][qb].x;
                            g.y -= a4[qa][qb].y;
                            G[row + col * ld] = g;
                        }
                    }
            }
        }
        grid.sync();
    }
    if (!info) {  // the strictly lower triangle is not part of R
        for (int64_t col = int64_t(c) * NW + warp; col < m; col += int64_t(NW) * ng)
            for (int64_t row = col + 1 + lane; row < m; row += 32) G[row + col * ld] = make_double2(0.0, 0.0);
    }
    if (c == 0) {
        // rank rule (src/solver.cpp:25-33, src/lsq.cpp:18-27) on the diagonal of R
        __shared__ double dstat[2];
        if (t == 0) {
            dstat[0] = dmin;
            dstat[1] = dmax;
        }
        __syncthreads();
        const double thr = rank_rows * kU * dstat[1];
        double bad = 0.0;
        if (!info)
            for (int64_t j = t; j < m; j += TH) {
                const double d = __ldcg(G + j + j * ld).x;
                if (d < thr || d == 0.0) bad += 1.0;
            }
        bad = block_sum(bad, red);
        if (t == 0) {
            st->info = info;
            st->deficient = int(bad);
            st->dmin = dstat[0];
            st->dmax = dstat[1];
            st->trace = tr;
            st->shift = shift;
            st->xnorm2 = 0.0;
        }
    }
}

// The Cholesky that produced R failed, or the diagonal ratio of R says u cond^2 > 1e-3 (the host
// then takes the shifted factorization, solver.cu cholqr_r): the stages queued behind it skip.
__device__ __forceinline__ bool chol_unusable(const CholStatus* st) {
    const int info = __ldcg(&st->info);
    const double dmin = __ldcg(&st->dmin), dmax = __ldcg(&st->dmax);
    if (info != 0 || !(dmin > 0.0)) return true;
    const double ratio = dmax / dmin;
    return kU * ratio * ratio > 1e-3;
}

// ------------------------------------------------------ triangular inverse
__global__ void __launch_bounds__(TH, 1)
trtri_upper_kernel(const double2* R, int64_t ldr, int64_t m, double2* X, double2* W, CholStatus* st, double* part,
                   int gate) {
    cg::grid_group grid = cg::this_grid();
    if (gate && chol_unusable(st)) return;  // (uniform: every CTA reads the same record)
    extern __shared__ double2 smem[];
    double2* D = smem;              // [NB][LDD]
    double2* As = D + NB * LDD;     // [KC][LDT]  (level 0: the inverse block, [NB][LDD])
    double2* Bs = As + KC * LDT;
    __shared__ double red[NW];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int ng = gridDim.x, c = blockIdx.x;
    const int64_t nblk = (m + NB - 1) / NB;

    // below the diagonal blocks X is zero
    for (int64_t col = int64_t(c) * NW + warp; col < m; col += int64_t(NW) * ng)
        for (int64_t row = (col / NB + 1) * NB + lane; row < m; row += 32) X[row + col * m] = make_double2(0.0, 0.0);

    // level 0: the diagonal blocks, a warp per column (lane i holds X[i, col])
    for (int64_t blk = c; blk < nblk; blk += ng) {
        const int64_t k0 = blk * NB;
        const int nb = int(imin64(NB, m - k0));
        __syncthreads();
        for (int e = t; e < NB * NB; e += TH) {
            const int i = e % NB, j = e / NB;
            D[i * LDD + j] = (i <= j && j < nb) ? R[(k0 + i) + (k0 + j) * ldr] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        for (int cc = warp; cc < nb; cc += NW) {
            double2 x = make_double2(0.0, 0.0);
            if (lane == cc) x = crecip(D[cc * LDD + cc]);
            for (int i = cc - 1; i >= 0; --i) {
                double2 p = make_double2(0.0, 0.0);
                if (lane > i && lane <= cc) cmac(p, D[i * LDD + lane], x);
                p = warp_sum2(p);
                if (lane == i) {
                    const double2 ri = crecip(D[i * LDD + i]);
                    x = make_double2(-(p.x * ri.x - p.y * ri.y), -(p.x * ri.y + p.y * ri.x));
                }
            }
            As[lane * LDD + cc] = lane <= cc ? x : make_double2(0.0, 0.0);
        }
        __syncthreads();
        for (int e = t; e < NB * NB; e += TH) {
            const int i = e % NB, j = e / NB;
            if (i < nb && j < nb) X[(k0 + i) + (k0 + j) * m] = As[i * LDD + j];
        }
    }
    grid.sync();

    // doubling levels: X12 = -X11 (R12 X22) for every aligned pair of s x s diagonal blocks
    const int tr_ = t & 15, tc_ = t >> 4;
    for (int64_t s = NB; s < m; s *= 2) {
        const int64_t span = 2 * s, npairs = (m + span - 1) / span;
        const int tI = int((s + TB - 1) / TB);
        const int64_t total = npairs * tI * tI;
        for (int phase = 0; phase < 2; ++phase) {
            for (int64_t tile = c; tile < total; tile += ng) {
                const int64_t p = tile / (tI * tI);
                const int rem = int(tile % (tI * tI)), ti = rem % tI, tj = rem / tI;
                const int64_t a = p * span;
                const int64_t s2 = imin64(s, m - a - s);
                const int64_t r0 = int64_t(ti) * TB, c0 = int64_t(tj) * TB;
                if (s2 <= 0 || c0 >= s2 || r0 >= s) continue;  // (uniform per CTA)
                const int rv = int(imin64(TB, s - r0)), cv = int(imin64(TB, s2 - c0));
                double2 a4[4][4];
                zero_acc(a4);
                double2* out;
                double sign;
                if (phase == 0) {  // W12 = R12 X22 (X22 upper: k <= j)
                    tile_mm<false>(R + (a + r0) + (a + s) * ldr, ldr, X + (a + s) + (a + s + c0) * m, m, 0,
                                   int(imin64(s2, c0 + TB)), rv, cv, As, Bs, a4);
                    out = W;
                    sign = 1.0;
                } else {           // X12 = -X11 W12 (X11 upper: k >= i)
                    tile_mm<false>(X + (a + r0) + a * m, m, W + a + (a + s + c0) * m, m, int(r0), int(s), rv, cv, As,
                                   Bs, a4);
                    out = X;
                    sign = -1.0;
                }
#pragma unroll
                for (int qa = 0; qa < 4; ++qa)
#pragma unroll
                    for (int qb = 0; qb < 4; ++qb) {
                        const int i = tr_ + 16 * qa, j = tc_ + 16 * qb;
                        if (i < rv && j < cv)
                            out[(a + r0 + i) + (a + s + c0 + j) * m] =
                                make_double2(sign * a4[qa][qb].x, sign * a4[qa][qb].y);
                    }
            }
            grid.sync();
        }
    }
    if (st) {  // ||X||_F^2 in a fixed order: per-CTA partials, then CTA 0
        double acc = 0.0;
        for (int64_t col = int64_t(c) * NW + warp; col < m; col += int64_t(NW) * ng)
            for (int64_t row = lane; row <= col; row += 32) {
                const double2 v = __ldcg(X + row + col * m);
                acc = fma(v.x, v.x, fma(v.y, v.y, acc));
            }
        acc = block_sum(acc, red);
        if (t == 0) part[c] = acc;
        grid.sync();
        if (c == 0) {
            double s2 = 0.0;
            for (int q = t; q < ng; q += TH) s2 += __ldcg(part + q);
            s2 = block_sum(s2, red);
            if (t == 0) st->xnorm2 = s2;
        }
    }
}

// ------------------------------------------------------ refinement loops
// y[j] = (base ? base[j] : 0) -/+ sum_r conj(M[r + j ld]) x[r]: a warp per column; tri: r <= j
__device__ __forceinline__ void gemv_cols_conj(const double2* M, int64_t ld, int64_t rows, int64_t cols, bool tri,
                                               const double2* x, const double2* base, double2* y) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t j = int64_t(blockIdx.x) * NW + warp; j < cols; j += int64_t(NW) * gridDim.x) {
        const int64_t nr = tri ? j + 1 : rows;
        const double2* col = M + j * ld;
        double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
        int64_t r = lane;
        for (; r + 96 < nr; r += 128) {
            cmac_conj(a0, __ldcg(col + r), __ldcg(x + r));
            cmac_conj(a1, __ldcg(col + r + 32), __ldcg(x + r + 32));
            cmac_conj(a2, __ldcg(col + r + 64), __ldcg(x + r + 64));
            cmac_conj(a3, __ldcg(col + r + 96), __ldcg(x + r + 96));
        }
        for (; r < nr; r += 32) cmac_conj(a0, __ldcg(col + r), __ldcg(x + r));
        double2 acc = make_double2((a0.x + a1.x) + (a2.x + a3.x), (a0.y + a1.y) + (a2.y + a3.y));
        acc = warp_sum2(acc);
        if (lane == 0) y[j] = base ? make_double2(base[j].x - acc.x, base[j].y - acc.y) : acc;
    }
}

// out[r] (+)= sum_j M[r + j ld] x_sh[j] over tasks of 32 rows (lanes = rows, the CTA's warps
// split the columns; fixed-order combine); tri: j >= the task's first row (M upper triangular).
// part (optional): part[task] = sum over the task's rows of |out[r]|^2.
__device__ __forceinline__ void gemv_rows(const double2* M, int64_t ld, int64_t rows, int64_t cols, bool tri,
                                          const double2* x_sh, double2* out, bool accumulate, double* part,
                                          double2 (*wp)[32]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntasks = (rows + 31) / 32;
    for (int64_t task = blockIdx.x; task < ntasks; task += gridDim.x) {
        const int64_t r = task * 32 + lane;
        const int64_t jlo = tri ? task * 32 : 0;
        const int64_t per = (cols - jlo + NW - 1) / NW;
        const int64_t j0 = jlo + warp * per, j1 = imin64(cols, j0 + per);
        double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
        if (r < rows) {
            const double2* row = M + r;
            int64_t j = j0;
            for (; j + 3 < j1; j += 4) {
                cmac(a0, __ldcg(row + j * ld), x_sh[j]);
                cmac(a1, __ldcg(row + (j + 1) * ld), x_sh[j + 1]);
                cmac(a2, __ldcg(row + (j + 2) * ld), x_sh[j + 2]);
                cmac(a3, __ldcg(row + (j + 3) * ld), x_sh[j + 3]);
            }
            for (; j < j1; ++j) cmac(a0, __ldcg(row + j * ld), x_sh[j]);
        }
        __syncthreads();
        wp[warp][lane] = make_double2((a0.x + a1.x) + (a2.x + a3.x), (a0.y + a1.y) + (a2.y + a3.y));
        __syncthreads();
        if (warp == 0) {
            double2 v = wp[0][lane];
#pragma unroll
            for (int q = 1; q < NW; ++q) {
                v.x += wp[q][lane].x;
                v.y += wp[q][lane].y;
            }
            double nrm = 0.0;
            if (r < rows) {
                if (accumulate) {
                    const double2 o = __ldcg(out + r);
                    v.x += o.x;
                    v.y += o.y;
                }
                out[r] = v;
                nrm = fma(v.x, v.x, v.y * v.y);
            }
            nrm = warp_sum1(nrm);
            if (part && lane == 0) part[task] = nrm;
        }
    }
}

// ||v||^2 of a global vector, the same fixed-order sum in every CTA
__device__ __forceinline__ double norm2_rep(const double2* v, int64_t len, double* red) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += TH) {
        const double2 e = __ldcg(v + i);
        acc = fma(e.x, e.x, fma(e.y, e.y, acc));
    }
    return block_sum(acc, red);
}
__device__ __forceinline__ double sum_rep(const double* v, int64_t len, double* red) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += TH) acc += __ldcg(v + i);
    return block_sum(acc, red);
}
__device__ __forceinline__ void load_vec(double2* sh, const double2* g, int64_t len) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < len; i += TH) sh[i] = __ldcg(g + i);
    __syncthreads();
}

__global__ void __launch_bounds__(TH, 1) sketch_refine_kernel(const RefineArgs p) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double2 smem[];
    double2* x_sh = smem;          // m: the input vector of the row products
    double2* v_sh = smem + p.m;    // m: PRECOND's unit vector (replicated)
    __shared__ double2 wp[NW][32];
    __shared__ double red[NW];
    const int64_t l = p.l, m = p.m;
    const int64_t ztasks = (l + 31) / 32;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (chol_unusable(p.chol)) {
        if (lead) {
            p.st->accepted = 0;
            p.st->iterations = 0;
            p.st->frobenius_ok = 0;
            p.st->best = 0.0;
            p.st->nz_best = 0.0;
            p.st->thr = 0.0;
        }
        return;
    }

    if (p.mode == REFINE_CSNE) {
        // z_0 = S G^{-1} b, z_{k+1} = z_k + S G^{-1} (b - S^H z_k), G^{-1} = X X^H, until the residual
        // stops halving; accepted at the rounding level 2 sqrt(l) u ||S||_F ||z||  (solver.cu step2)
        const double thr = 2.0 * sqrt(double(l)) * kU * sqrt(fmax(__ldcg(&p.chol->trace), 0.0));
        double prev = 0.0, best = 0.0, nz_best = 0.0;
        int its = 0;
        const double2* w = p.b;  // the right-hand side of the next G^{-1} solve
        for (int it = -1; it <= 6; ++it) {
            if (it >= 0) {
                gemv_cols_conj(p.S, l, l, m, false, p.z, p.b, p.v0);  // w = b - S^H z
                grid.sync();
                const double nr = sqrt(norm2_rep(p.v0, m, red));
                const double nz = sqrt(sum_rep(p.part, ztasks, red));
                if (lead && it < 8) p.st->resid[it] = nr;
                if (it == 0 || nr < best) {
                    best = nr;
                    nz_best = nz;
                }
                its = it;
                if (nr == 0.0) break;
                if ((it > 0 && !(nr < 0.5 * prev)) || it == 6) break;
                prev = nr;
                w = p.v0;
            }
            gemv_cols_conj(p.X, m, m, m, true, w, nullptr, p.v1);      // X^H w
            grid.sync();
            load_vec(x_sh, p.v1, m);
            gemv_rows(p.X, m, m, m, true, x_sh, p.v2, false, nullptr, wp);  // X (X^H w)
            grid.sync();
            load_vec(x_sh, p.v2, m);
            gemv_rows(p.S, l, l, m, false, x_sh, p.z, it >= 0, p.part, wp);  // z (+)= S (...)
            grid.sync();
        }
        if (lead) {
            p.st->accepted = (best == 0.0 || best <= thr * nz_best) ? 1 : 0;
            p.st->iterations = its;
            p.st->frobenius_ok = 0;
            p.st->best = best;
            p.st->nz_best = nz_best;
            p.st->thr = thr;
        }
        return;
    }

    // PRECOND: one Cholesky pass is enough when Q1 = E X is orthonormal to 1e-3 (solver.cu
    // cholqr_r): the free bound u ||R1||_F^2 ||X||_F^2 first, else power steps on D = Q1^H Q1 - I
    const double bound = kU * __ldcg(&p.chol->trace) * __ldcg(&p.chol->xnorm2);
    const bool frob = bound <= 1e-3;
    if (frob || !p.two_norm_check) {
        if (lead) {
            p.st->accepted = frob ? 1 : 0;
            p.st->iterations = 0;
            p.st->frobenius_ok = frob ? 1 : 0;
            p.st->best = 0.0;
            p.st->nz_best = 0.0;
            p.st->thr = bound;
        }
        return;
    }
    for (int64_t i = threadIdx.x; i < m; i += TH) v_sh[i] = p.b[i];
    double nrm = sqrt(norm2_rep(p.b, m, red));
    for (int it = 0; it < p.power_steps; ++it) {
        __syncthreads();
        const double inv = 1.0 / nrm;
        for (int64_t i = threadIdx.x; i < m; i += TH) v_sh[i] = make_double2(v_sh[i].x * inv, v_sh[i].y * inv);
        __syncthreads();
        gemv_rows(p.X, m, m, m, true, v_sh, p.v1, false, nullptr, wp);   // a = X v
        grid.sync();
        load_vec(x_sh, p.v1, m);
        gemv_rows(p.S, l, l, m, false, x_sh, p.z, false, nullptr, wp);   // q = E a
        grid.sync();
        gemv_cols_conj(p.S, l, l, m, false, p.z, nullptr, p.v2);         // a = E^H q
        grid.sync();
        gemv_cols_conj(p.X, m, m, m, true, p.v2, nullptr, p.v0);         // q = X^H a
        grid.sync();
        double acc = 0.0;
        for (int64_t i = threadIdx.x; i < m; i += TH) {                  // v = D v
            const double2 q = __ldcg(p.v0 + i);
            const double2 d = make_double2(q.x - v_sh[i].x, q.y - v_sh[i].y);
            v_sh[i] = d;
            acc = fma(d.x, d.x, fma(d.y, d.y, acc));
        }
        nrm = sqrt(block_sum(acc, red));
        if (nrm == 0.0) break;
    }
    if (lead) {
        p.st->accepted = 2.0 * nrm <= 1e-3 ? 1 : 0;
        p.st->iterations = p.power_steps;
        p.st->frobenius_ok = 0;
        p.st->best = nrm;
        p.st->nz_best = 0.0;
        p.st->thr = bound;
    }
}

// Rank rule (src/solver.cpp:25-33, src/lsq.cpp:18-27) on the diagonal of R = R2 R1 (both upper
// triangular with positive diagonals, so R_jj = R2_jj R1_jj): st->deficient.  One CTA.
__global__ void __launch_bounds__(TH, 1)
diag_product_rank_kernel(const double2* R2, int64_t ld2, const double2* R1, int64_t ld1, int64_t m, double rows,
                         CholStatus* st) {
    __shared__ double red[NW];
    double dmax = 0.0;
    for (int64_t j = threadIdx.x; j < m; j += TH)
        dmax = fmax(dmax, fabs(__ldcg(R2 + j + j * ld2).x) * fabs(__ldcg(R1 + j + j * ld1).x));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
    __syncthreads();
    dmax = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) dmax = fmax(dmax, red[q]);
    const double thr = rows * kU * dmax;
    double bad = 0.0;
    for (int64_t j = threadIdx.x; j < m; j += TH) {
        const double d = fabs(__ldcg(R2 + j + j * ld2).x) * fabs(__ldcg(R1 + j + j * ld1).x);
        if (d < thr || d == 0.0) bad += 1.0;
    }
    bad = block_sum(bad, red);
    if (threadIdx.x == 0) st->deficient = int(bad);
}

constexpr size_t kTileSmem = size_t(NB * LDD + 2 * KC * LDT) * sizeof(double2);
constexpr size_t kCholSmem = kTileSmem + size_t(NB * LDD) * sizeof(double2);

}  // namespace

int chol_grid(int64_t m, int num_sms) {
    const int64_t nt = (std::max<int64_t>(m - NB, 0) + TB - 1) / TB;
    const int64_t tiles = nt * (nt + 1) / 2;
    // enough CTAs for the first trailing update's tiles and for one panel column per warp
    const int64_t panel = (std::max<int64_t>(m - NB, 0) + NW - 1) / NW;
    return int(std::max<int64_t>(1, std::min<int64_t>(num_sms, std::max<int64_t>(tiles, panel))));
}

void launch_chol_upper(double2* G, int64_t m, int64_t ld, double shift_factor, double rank_rows, CholStatus* st,
                       int num_sms, cudaStream_t stream) {
    auto k = chol_upper_kernel;
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCholSmem)));
    void* params[] = {&G, &m, &ld, &shift_factor, &rank_rows, &st};
    MNB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(chol_grid(m, num_sms)), dim3(TH),
                                         params, kCholSmem, stream));
}

void launch_trtri_upper(const double2* R, int64_t ldr, int64_t m, double2* X, double2* W, CholStatus* st,
                        int num_sms, cudaStream_t stream, bool gate_on_chol) {
    auto k = trtri_upper_kernel;
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTileSmem)));
    const int64_t top = (m + 127) / 128;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(num_sms, std::max<int64_t>((m + NB - 1) / NB, top * top))));
    // the per-CTA partials of ||X||_F^2 live at the head of W's last column block: W is only
    // written in columns >= 32 (every W12 sits right of a diagonal block), its first column is free
    double* part = reinterpret_cast<double*>(W);
    int gate = gate_on_chol && st ? 1 : 0;
    void* params[] = {&R, &ldr, &m, &X, &W, &st, &part, &gate};
    MNB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(TH), params, kTileSmem,
                                         stream));
}

void launch_diag_product_rank(const double2* R2, int64_t ld2, const double2* R1, int64_t ld1, int64_t m, double rows,
                              CholStatus* st, cudaStream_t stream) {
    diag_product_rank_kernel<<<1, TH, 0, stream>>>(R2, ld2, R1, ld1, m, rows, st);
    MNB_LAUNCH_CHECK();
}

void launch_sketch_refine(const RefineArgs& a, int num_sms, cudaStream_t stream) {
    auto k = sketch_refine_kernel;
    const size_t smem = size_t(2 * a.m) * sizeof(double2);
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int grid = int(std::max<int64_t>(
        1, std::min<int64_t>(num_sms, std::max<int64_t>((a.l + 31) / 32, (a.m + NW - 1) / NW))));
    RefineArgs args = a;
    void* params[] = {&args};
    MNB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(TH), params, smem, stream));
}

}  // namespace mnb
