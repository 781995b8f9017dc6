// Batched FP64 FFT passes over rows of a column-major block (sm_100a).
//
// Replaces the reference's per-row radix-2 / Bluestein Fft::forward
// (src/fft.cpp:65-97) inside the SRFT sketch.  A length-n transform is a
// four-step n = n1*n2 (two launches: pass A = length-n2 DFTs over the
// stride-n1 sub-sequences with the w_n^{f2 k1} twiddle fused into the
// epilogue, pass B = length-n1 DFTs whose epilogue keeps only the l sampled
// frequencies, src/srft.cpp:131), or a single launch for n <= 2048.
//
// One CTA = Rb rows x one length-N sub-transform.  Each thread keeps E
// elements in registers; a pass of radix R (R | E) is E/R register
// butterflies; passes exchange data through shared memory in place (all
// reads, barrier, all writes).  Mixed-radix Stockham ordering, so the output
// is in natural order with no bit reversal.  Radices 16, 8, 4, 3, 2.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "fft_dev.cuh"

namespace mnb {

namespace {

template <int R, bool INV>
__device__ __forceinline__ void dft_r(double2* x) {
    if constexpr (R == 2) dft2<INV>(x[0], x[1]);
    else if constexpr (R == 3) dft3<INV>(x[0], x[1], x[2]);
    else if constexpr (R == 4) dft4<INV>(x[0], x[1], x[2], x[3]);
    else if constexpr (R == 8) dft8<INV>(x);
    else if constexpr (R == 16) dft16<INV>(x);
}

__device__ __forceinline__ double2 tw_at(const double2* __restrict__ tw, int64_t q, bool inv) {
    double2 w = __ldg(tw + q);
    if (inv) w.y = -w.y;
    return w;
}

__device__ __forceinline__ uint32_t sm_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tile_load(double2* dst, const double2* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sm_u32(dst)),
                 "l"(src), "r"(bytes), "r"(sm_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tile_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(sm_u32(bar)), "r"(parity)
            : "memory");
    }
}

// Load phase helper: first pass reads global, later passes read shared.
template <int Rb, int E, bool INV>
struct FftCta {
    const FftPassArgs& a;
    double2* sm;
    int r, u, U;
    int64_t row, b;
    bool row_ok;
    int64_t rbk = 0;                     // blocked mode: row block of this unit
    uint64_t* bar = nullptr;             // blocked mode: tile mbarrier
    const double2* next_tile = nullptr;  // blocked mode: tile to prefetch once the last pass has read smem
    uint32_t tile_bytes = 0;

    __device__ __forceinline__ double2 gload(int idx) const {
        if (!row_ok) return make_double2(0.0, 0.0);
        if (a.blocked)  // tile of unit (row block, b) is [N][8] at in + ((row/8)*batches + b)*N*8
            return __ldg(a.in + (((row >> 3) * a.batches + b) * a.N + idx) * 8 + (row & 7));
        const int64_t col = b * a.in_bstride + int64_t(idx) * a.in_istride;
        return __ldg(a.in + (a.in_row0 + row) + col * a.ld_in);
    }

    __device__ __forceinline__ void gstore(int f, double2 v) const {
        if (!row_ok) return;
        if (a.mode == FFT_OUT_TWIDDLE) {
            const int64_t e = int64_t(f) * b;  // f < n2, b < n1: already below n
            double2 w = c_mul(__ldg(a.tw4_hi + (e >> a.tw4_shift)), __ldg(a.tw4_lo + (e & ((int64_t(1) << a.tw4_shift) - 1))));
            if (INV) w.y = -w.y;
            v = c_mul(v, w);
            if (a.blocked) {  // [row block][f][b][8]: the next pass reads one contiguous tile
                a.out[(((row >> 3) * a.N + f) * a.batches + b) * 8 + (row & 7)] = v;
                return;
            }
            const int64_t col = int64_t(f) * a.out_fstride + b * a.out_bstride;
            a.out[(a.out_row0 + row) + col * a.ld_out] = v;
        } else if (a.mode == FFT_OUT_SELECT) {
            const int64_t F = b + a.nb * int64_t(f);
            const int slot = __ldg(a.sel + F);
            if (slot >= 0) a.out[int64_t(slot) + (a.out_row0 + row) * a.ld_out] = c_scale(v, a.scale);
        } else {
            const int64_t col = b + a.nb * int64_t(f);
            a.out[(a.out_row0 + row) + col * a.ld_out] = c_scale(v, a.scale);
        }
    }

    template <int R>
    __device__ __forceinline__ void pass(double2 (&v)[E], int Ns, bool first, bool last) {
        constexpr int B = E / R;  // butterflies per thread
        const int N = a.N;
        const int NR = N / R;
        // read
#pragma unroll
        for (int s = 0; s < B; ++s) {
            const int j = u + s * U;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int idx = j + q * NR;
                v[s * R + q] = first ? gload(idx) : sm[idx * Rb + r];
            }
        }
        // twiddle + butterfly
        const int stride = N / (Ns * R);
#pragma unroll
        for (int s = 0; s < B; ++s) {
            const int j = u + s * U;
            const int k = j % Ns;
            if (k != 0) {
#pragma unroll
                for (int q = 1; q < R; ++q) v[s * R + q] = c_mul(v[s * R + q], tw_at(a.tw, int64_t(k) * q * stride, INV));
            }
            dft_r<R, INV>(&v[s * R]);
        }
        if (!first) __syncthreads();  // all in-place reads done before any write
        if (last && next_tile && threadIdx.x == 0) {  // blocked mode: the tile buffer is free -> prefetch
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tile_load(sm, next_tile, tile_bytes, bar);
        }
        // write
#pragma unroll
        for (int s = 0; s < B; ++s) {
            const int j = u + s * U;
            const int k = j % Ns;
            const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int o = idxD + q * Ns;
                if (last) gstore(o, v[s * R + q]);
                else sm[o * Rb + r] = v[s * R + q];
            }
        }
        if (!last) __syncthreads();
    }
};

template <int Rb, int E, bool INV>
__global__ void __launch_bounds__(512) fft_pass_kernel(const FftPassArgs a) {
    extern __shared__ double2 sm[];
    FftCta<Rb, E, INV> cta{a, sm, int(threadIdx.x % Rb), int(threadIdx.x / Rb), a.N / E, 0, 0, false};
    cta.row = int64_t(blockIdx.x) * Rb + cta.r;
    cta.row_ok = cta.row < a.rows;
    cta.b = blockIdx.y;
    double2 v[E];
    int Ns = 1;
    for (int p = 0; p < a.nradix; ++p) {
        const int R = a.radix[p];
        const bool first = p == 0, last = p == a.nradix - 1;
        switch (R) {
            case 2: if constexpr (E % 2 == 0) cta.template pass<2>(v, Ns, first, last); break;
            case 3: if constexpr (E % 3 == 0) cta.template pass<3>(v, Ns, first, last); break;
            case 4: if constexpr (E % 4 == 0) cta.template pass<4>(v, Ns, first, last); break;
            case 8: if constexpr (E % 8 == 0) cta.template pass<8>(v, Ns, first, last); break;
            case 16: if constexpr (E % 16 == 0) cta.template pass<16>(v, Ns, first, last); break;
            default: break;
        }
        Ns *= R;
    }
}

// Blocked four-step pass: unit (row block rbk of 8 rows, batch b) reads ONE
// contiguous tile [N][8] (in + (rbk*batches + b)*N*8) with a TMA bulk copy,
// so HBM sees 128 KiB sequential reads instead of N scattered 128-byte pieces.
//
// Persistent CTAs, N/2 threads (E = 16 elements each, the whole tile in
// registers).  Shared memory = the tile buffer + a half-tile exchange buffer:
//   wait tile -> registers -> barrier -> prefetch the NEXT tile into the
//   buffer (TMA, overlapping every radix pass and the global stores of this
//   unit) -> radix passes in registers; between passes the data is exchanged
//   through the half buffer one 4-row half at a time (rows are independent
//   transforms) -> the last pass stores to global (twiddled, blocked for the
//   next pass, or the sampled frequencies).
template <int E, bool INV>
struct FftTile {
    static constexpr int Rb = 8;
    const FftPassArgs& a;
    FftCta<Rb, E, INV>& cta;  // epilogue (gstore) and twiddle table
    const int N, U, r, u;

    // inputs of a radix-R pass: v[s*R + q] = x[u + s*U + q*N/R]
    template <int R, class Src>
    __device__ __forceinline__ void load(double2 (&v)[E], Src src) const {
        constexpr int B = E / R;
        const int NR = N / R;
#pragma unroll
        for (int s = 0; s < B; ++s)
#pragma unroll
            for (int q = 0; q < R; ++q) v[s * R + q] = src(u + s * U + q * NR);
    }
    template <int R>
    __device__ __forceinline__ void compute(double2 (&v)[E], int Ns) const {
        constexpr int B = E / R;
        const int stride = N / (Ns * R);
#pragma unroll
        for (int s = 0; s < B; ++s) {
            const int j = u + s * U;
            const int k = j % Ns;
            if (k != 0) {
#pragma unroll
                for (int q = 1; q < R; ++q) v[s * R + q] = c_mul(v[s * R + q], tw_at(a.tw, int64_t(k) * q * stride, INV));
            }
            dft_r<R, INV>(&v[s * R]);
        }
    }
    // outputs of a radix-R pass: y[(j/Ns)*Ns*R + j%Ns + q*Ns] = v[s*R + q]
    template <int R, class Dst>
    __device__ __forceinline__ void store(const double2 (&v)[E], int Ns, Dst dst) const {
        constexpr int B = E / R;
#pragma unroll
        for (int s = 0; s < B; ++s) {
            const int j = u + s * U;
            const int k = j % Ns;
            const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
            for (int q = 0; q < R; ++q) dst(idxD + q * Ns, v[s * R + q]);
        }
    }
};

template <int E, bool INV>
__global__ void __launch_bounds__(512, 1) fft_tile_kernel(const FftPassArgs a) {
    constexpr int Rb = 8;
    extern __shared__ double2 sm[];
    const int N = a.N;
    double2* T = sm;                          // tile [N][8]
    double2* X = sm + size_t(N) * Rb;         // exchange [N][4]
    uint64_t* bar = reinterpret_cast<uint64_t*>(X + size_t(N) * 4);
    const int r = int(threadIdx.x % Rb), u = int(threadIdx.x / Rb), U = N / E;
    FftCta<Rb, E, INV> cta{a, sm, r, u, U, 0, 0, false};
    const FftTile<E, INV> ft{a, cta, N, U, r, u};
    const int64_t nrbk = (a.rows + Rb - 1) / Rb;
    const int64_t units = nrbk * a.batches;
    const int64_t tile = int64_t(N) * Rb;
    const uint32_t tile_bytes = uint32_t(tile * 16);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int64_t unit = blockIdx.x;
    if (threadIdx.x == 0 && unit < units) tile_load(T, a.in + unit * tile, tile_bytes, bar);
    uint32_t phase = 0;
    double2 v[E];
    const int half = r >> 2, r4 = r & 3;
    for (; unit < units; unit += gridDim.x) {
        cta.rbk = unit / a.batches;
        cta.b = unit - cta.rbk * a.batches;
        cta.row = cta.rbk * Rb + r;
        cta.row_ok = cta.row < a.rows;
        tile_wait(bar, phase);
        phase ^= 1u;
        auto from_tile = [&](int idx) { return T[idx * Rb + r]; };
        switch (a.radix[0]) {
            case 16: if constexpr (E % 16 == 0) ft.template load<16>(v, from_tile); break;
            case 8: if constexpr (E % 8 == 0) ft.template load<8>(v, from_tile); break;
            case 4: if constexpr (E % 4 == 0) ft.template load<4>(v, from_tile); break;
            case 3: if constexpr (E % 3 == 0) ft.template load<3>(v, from_tile); break;
            default: if constexpr (E % 2 == 0) ft.template load<2>(v, from_tile); break;
        }
        __syncthreads();  // the tile buffer is free: fetch the next unit's tile behind the compute
        const int64_t next = unit + gridDim.x;
        if (threadIdx.x == 0 && next < units) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tile_load(T, a.in + next * tile, tile_bytes, bar);
        }
        int Ns = 1;
        for (int p = 0; p < a.nradix; ++p) {
            const int R = a.radix[p];
            const bool last = p == a.nradix - 1;
            auto to_global = [&](int o, double2 val) { cta.gstore(o, val); };
            auto to_x = [&](int o, double2 val) { X[o * 4 + r4] = val; };
            auto from_x = [&](int idx) { return X[idx * 4 + r4]; };
#define MNB_TILE_STEP(RR)                                                          \
    if constexpr (E % RR == 0) {                                                   \
        ft.template compute<RR>(v, Ns);                                            \
        if (last) {                                                                \
            ft.template store<RR>(v, Ns, to_global);                               \
        } else {                                                                   \
            for (int h = 0; h < 2; ++h) {                                          \
                if (half == h) ft.template store<RR>(v, Ns, to_x);                 \
                __syncthreads();                                                   \
                if (half == h) {                                                   \
                    switch (a.radix[p + 1]) {                                      \
                        case 16: if constexpr (E % 16 == 0) ft.template load<16>(v, from_x); break; \
                        case 8: if constexpr (E % 8 == 0) ft.template load<8>(v, from_x); break;    \
                        case 4: if constexpr (E % 4 == 0) ft.template load<4>(v, from_x); break;    \
                        case 3: if constexpr (E % 3 == 0) ft.template load<3>(v, from_x); break;    \
                        default: if constexpr (E % 2 == 0) ft.template load<2>(v, from_x); break;   \
                    }                                                              \
                }                                                                  \
                __syncthreads();                                                   \
            }                                                                      \
        }                                                                          \
    }
            switch (R) {
                case 16: MNB_TILE_STEP(16) break;
                case 8: MNB_TILE_STEP(8) break;
                case 4: MNB_TILE_STEP(4) break;
                case 3: MNB_TILE_STEP(3) break;
                default: MNB_TILE_STEP(2) break;
            }
#undef MNB_TILE_STEP
            Ns *= R;
        }
    }
}

// Specialised N = 1024 blocked pass (radix 16 x 16 x 4, forward): the
// structure of fft_tile_kernel with every stride a compile-time constant, the
// length-1024 twiddles in shared memory, and the epilogue data of the unit
// (four-step twiddles w_n^{f b}, or the frequency -> sample-slot map) gathered
// into shared memory while pass 1 computes, so no global load sits on the
// store path.  512 threads: row r = tid & 7, u = tid >> 3 (64 threads per row,
// 16 elements each).
template <bool SELECT>
__global__ void __launch_bounds__(512, 1) fft1024_tile_kernel(const FftPassArgs a) {
    constexpr int Rb = 8, N = 1024;
    extern __shared__ double2 sm[];
    double2* T = sm;             // tile [1024][8]   128 KiB
    double2* X = T + N * Rb;     // exchange [1024][4]  64 KiB
    double2* W = X + N * 4;      // w_1024^k           16 KiB
    double2* Z = W + N;          // epilogue data of the unit (16 KiB)
    int* Zs = reinterpret_cast<int*>(Z);
    uint64_t* bar = reinterpret_cast<uint64_t*>(Z + N);
    const int r = int(threadIdx.x & 7), u = int(threadIdx.x >> 3);
    const int half = r >> 2, r4 = r & 3;
    const int64_t nrbk = (a.rows + Rb - 1) / Rb;
    const int64_t units = nrbk * a.batches;
    constexpr int64_t tile = int64_t(N) * Rb;
    constexpr uint32_t tile_bytes = uint32_t(tile * 16);
    for (int i = threadIdx.x; i < N; i += blockDim.x) W[i] = __ldg(a.tw + i);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int64_t unit = blockIdx.x;
    if (threadIdx.x == 0 && unit < units) tile_load(T, a.in + unit * tile, tile_bytes, bar);
    uint32_t phase = 0;
    const int64_t lo_mask = (int64_t(1) << a.tw4_shift) - 1;
#define XI(o) (((o) << 2) + r4)
    double2 v[16];
    for (; unit < units; unit += gridDim.x) {
        const int64_t rbk = unit / a.batches, b = unit - rbk * a.batches;
        const int64_t row = rbk * Rb + r;
        // epilogue data for frequencies f = tid, tid + 512 (loads in flight during the tile wait and pass 1)
        double2 zt[2];
        int zs[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int64_t f = threadIdx.x + 512 * i;
            if constexpr (SELECT) {
                zs[i] = __ldg(a.sel + b + a.nb * f);
            } else {
                const int64_t e = f * b;  // < n
                zt[i] = c_mul(__ldg(a.tw4_hi + (e >> a.tw4_shift)), __ldg(a.tw4_lo + (e & lo_mask)));
            }
        }
        tile_wait(bar, phase);
        phase ^= 1u;
        // pass 1 (radix 16, Ns = 1): x[u + 64 q]
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = T[(u + 64 * q) * Rb + r];
        __syncthreads();  // tile buffer free (and the previous unit's epilogue done with Z)
        {
            const int64_t next = unit + gridDim.x;
            if (threadIdx.x == 0 && next < units) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tile_load(T, a.in + next * tile, tile_bytes, bar);
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            if constexpr (SELECT) Zs[threadIdx.x + 512 * i] = zs[i];
            else Z[threadIdx.x + 512 * i] = zt[i];
        }
        dft16_np<false>(v);
        // -> y[16 u + q];   pass 2 (radix 16, Ns = 16) reads x[u + 64 q], twiddle w^{4 (u%16) q}
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (half == h) {
#pragma unroll
                for (int q = 0; q < 16; ++q) X[XI(16 * u + q)] = v[d16(q)];
            }
            __syncthreads();
            if (half == h) {
#pragma unroll
                for (int q = 0; q < 16; ++q) v[q] = X[XI(u + 64 * q)];
            }
            __syncthreads();
        }
        {
            const int k = u & 15;
#pragma unroll
            for (int q = 1; q < 16; ++q) v[q] = c_mul(v[q], W[4 * k * q]);
        }
        dft16_np<false>(v);
        // -> y[(u/16)*256 + u%16 + 16 q];   pass 3 (radix 4, Ns = 256) reads x[j + 256 q], j = u + 64 s
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (half == h) {
#pragma unroll
                for (int q = 0; q < 16; ++q) X[XI((u >> 4) * 256 + (u & 15) + 16 * q)] = v[d16(q)];
            }
            __syncthreads();
            if (half == h) {
#pragma unroll
                for (int s = 0; s < 4; ++s)
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[4 * s + q] = X[XI(u + 64 * s + 256 * q)];
            }
            __syncthreads();
        }
        const bool row_ok = row < a.rows;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int j = u + 64 * s;
#pragma unroll
            for (int q = 1; q < 4; ++q) v[4 * s + q] = c_mul(v[4 * s + q], W[j * q]);
            dft4<false>(v[4 * s], v[4 * s + 1], v[4 * s + 2], v[4 * s + 3]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int f = j + 256 * q;
                if constexpr (SELECT) {
                    const int slot = Zs[f];
                    if (slot >= 0 && row_ok) a.out[int64_t(slot) + (a.out_row0 + row) * a.ld_out] = c_scale(v[4 * s + q], a.scale);
                } else {
                    // blocked [row block][f][b][8] for pass B
                    a.out[((rbk * N + f) * a.batches + b) * Rb + r] = c_mul(v[4 * s + q], Z[f]);
                }
            }
        }
    }
#undef XI
}

// In-warp transposed reduction of 4 values: afterwards lane l holds the warp-wide
// sum of value index l >> 3 in v[0] (3 + 3 shuffle rounds).
__device__ __forceinline__ void xreduce4(double (&v)[4], int lane) {
    {
        const bool up = (lane & 16) != 0;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double send = up ? v[i] : v[i + 2];
            const double keep = up ? v[i + 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
    }
    {
        const bool up = (lane & 8) != 0;
        const double send = up ? v[0] : v[1];
        const double keep = up ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
}

constexpr int kEnt = 512;  // staged (f1, slot) pairs per pass-B unit

// Pass B of the sketch FFT with N = n1 = 1024, pruned to the sampled outputs.
// Only ~l/n2 of the 1024 frequencies of a unit (row block rbk, f2 = b) are
// kept (src/srft.cpp:131), so after the first radix-16 stage,
//   Y_u[j] = sum_q x[u + 64 q] w_16^{j q}          (u < 64, j < 16),
// each kept frequency f is a 64-term sum  X[f] = sum_u w_1024^{f u} Y_u[f mod 16].
// Every thread (row r, u) holds its Y_u[j] in registers, so it forms its term
// of every kept sum directly; the 4 u of a warp are summed by shuffles and the
// 16 warps through a small shared partial table (fixed order: deterministic).
// No exchange of the transform.  The unit's samples come from a CSR list
// (off/ent: per f2 the pairs (f1, slot), sorted by f1 mod 16 on the host) so
// the register index j is a compile-time constant in the loop over j.
constexpr int kSB = 16;  // samples per partial-table batch

__global__ void __launch_bounds__(512, 1) fft1024_select_kernel(const FftPassArgs a, const int32_t* __restrict__ off,
                                                              const int32_t* __restrict__ ent) {
    constexpr int Rb = 8, N = 1024;
    extern __shared__ double2 sm[];
    double2* T = sm;                         // tile [1024][8]
    double2* W = T + N * Rb;                 // w_1024^k
    double2* P = W + N;                      // partial sums [16 warps][kSB][8 rows]
    int32_t* ENT = reinterpret_cast<int32_t*>(P + 16 * kSB * 8);  // the unit's (f1, slot) pairs, up to kEnt
    int32_t* JOFF = ENT + 2 * kEnt;          // first entry with f1 mod 16 >= j, j = 0..16
    uint64_t* bar = reinterpret_cast<uint64_t*>(JOFF + 20);
    const int r = int(threadIdx.x & 7), u = int(threadIdx.x >> 3);
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    const int64_t nrbk = (a.rows + Rb - 1) / Rb;
    const int64_t units = nrbk * a.batches;
    constexpr int64_t tile = int64_t(N) * Rb;
    constexpr uint32_t tile_bytes = uint32_t(tile * 16);
    for (int i = threadIdx.x; i < N; i += blockDim.x) W[i] = __ldg(a.tw + i);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int64_t unit = blockIdx.x;
    if (threadIdx.x == 0 && unit < units) tile_load(T, a.in + unit * tile, tile_bytes, bar);
    uint32_t phase = 0;
    double2 v[16];
    for (; unit < units; unit += gridDim.x) {
        const int64_t rbk = unit / a.batches, b = unit - rbk * a.batches;
        const int e0 = __ldg(off + b), cnt = __ldg(off + b + 1) - e0;
        const int32_t* E = cnt <= kEnt ? ENT : ent + 2 * e0;
        // the unit's sample list and its j ranges (read by every thread) while the tile lands
        for (int t = threadIdx.x; t < 2 * min(cnt, kEnt); t += blockDim.x) ENT[t] = __ldg(ent + 2 * e0 + t);
        if (threadIdx.x < 17) {
            int o = 0;
            while (o < cnt && (__ldg(ent + 2 * (e0 + o)) & 15) < int(threadIdx.x)) ++o;
            JOFF[threadIdx.x] = o;
        }
        tile_wait(bar, phase);
        phase ^= 1u;
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = T[(u + 64 * q) * Rb + r];
        __syncthreads();  // tile buffer free; ENT / JOFF visible
        {
            const int64_t next = unit + gridDim.x;
            if (threadIdx.x == 0 && next < units) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tile_load(T, a.in + next * tile, tile_bytes, bar);
            }
        }
        if (cnt == 0) continue;  // uniform; the next iteration's barrier orders the buffers' reuse
        dft16_np<false>(v);
        for (int b0 = 0; b0 < cnt; b0 += kSB) {
            const int nb = min(kSB, cnt - b0);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int lo = max(JOFF[j], b0), hi = min(JOFF[j + 1], b0 + nb);
                for (int s = lo; s < hi; ++s) {  // warp-uniform bounds: the shuffles are convergent
                    const int f = E[2 * s];
                    double2 p = c_mul(v[d16(j)], W[(f * u) & (N - 1)]);
#pragma unroll
                    for (int o = 8; o < 32; o <<= 1) {
                        p.x += __shfl_xor_sync(0xffffffffu, p.x, o);
                        p.y += __shfl_xor_sync(0xffffffffu, p.y, o);
                    }
                    if (lane < 8) P[(warp * kSB + (s - b0)) * 8 + lane] = p;
                }
            }
            __syncthreads();
            if (int(threadIdx.x) < 8 * nb) {
                const int rr = int(threadIdx.x) & 7, sl = int(threadIdx.x) >> 3;
                double2 acc = P[sl * 8 + rr];
#pragma unroll
                for (int w = 1; w < 16; ++w) acc = c_add(acc, P[(w * kSB + sl) * 8 + rr]);
                const int64_t row = rbk * Rb + rr;
                if (row < a.rows) a.out[int64_t(E[2 * (b0 + sl) + 1]) + (a.out_row0 + row) * a.ld_out] = c_scale(acc, a.scale);
            }
            if (b0 + kSB < cnt) __syncthreads();  // P reused by the next batch
        }
    }
}

// Pass B pruned to the sampled frequencies for the plain [n][Ms] layout and any
// N = 16 U (U <= 128; e.g. 2048 or 1536 at n = 3*2^20): Y_u[j] = sum_q
// x[u + U q] w_16^{j q} in registers (16 loads per thread straight from global,
// Rb rows x U threads), then each kept frequency is X[f] = sum_u w_N^{f u}
// Y_u[f mod 16], one warp per (row, sample) pair.  Persistent over units
// (row block, f2); the next unit's loads are issued before the warp sums.
__global__ void __launch_bounds__(512, 1) fft_select_pruned_kernel(const FftPassArgs a, const int32_t* __restrict__ off,
                                                                 const int32_t* __restrict__ ent, int Rb, int U) {
    extern __shared__ double2 sm[];
    const int N = a.N;
    double2* W = sm;          // w_N^k
    double2* X = sm + N;      // [Rb][16][U]
    const int r = int(threadIdx.x) % Rb, u = int(threadIdx.x) / Rb;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31), nwarps = int(blockDim.x >> 5);
    for (int i = threadIdx.x; i < N; i += blockDim.x) W[i] = __ldg(a.tw + i);
    const int64_t nrb = (a.rows + Rb - 1) / Rb;
    const int64_t units = nrb * a.batches;
    auto load = [&](int64_t unit, double2 (&v)[16]) {
        const int64_t rb = unit / a.batches, b = unit - rb * a.batches;
        const int64_t row = rb * Rb + r;
        if (row >= a.rows) {
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = make_double2(0.0, 0.0);
            return;
        }
        const double2* base = a.in + (a.in_row0 + row) + b * a.in_bstride * a.ld_in;
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = __ldg(base + int64_t(u + U * q) * a.in_istride * a.ld_in);
    };
    double2 v[16];
    int64_t unit = blockIdx.x;
    if (unit < units) load(unit, v);
    for (; unit < units; unit += gridDim.x) {
        const int64_t rb = unit / a.batches, b = unit - rb * a.batches;
        dft16_np<false>(v);
        __syncthreads();  // the previous unit's sums are done with X (and W is loaded)
#pragma unroll
        for (int j = 0; j < 16; ++j) X[(r * 16 + j) * U + u] = v[d16(j)];
        __syncthreads();
        const int64_t next = unit + gridDim.x;
        if (next < units) load(next, v);  // in flight during the sums
        const int e0 = __ldg(off + b), cnt = __ldg(off + b + 1) - e0;
        for (int p = warp; p < Rb * cnt; p += nwarps) {
            const int rp = p % Rb, s = p / Rb;
            const int f = __ldg(ent + 2 * (e0 + s)), slot = __ldg(ent + 2 * (e0 + s) + 1);
            const double2* Y = X + (rp * 16 + (f & 15)) * U;
            double2 acc = make_double2(0.0, 0.0);
            for (int uu = lane; uu < U; uu += 32) {
                const double2 y = Y[uu];
                const double2 w = W[(int64_t(f) * uu) % N];
                acc.x = fma(y.x, w.x, fma(-y.y, w.y, acc.x));
                acc.y = fma(y.x, w.y, fma(y.y, w.x, acc.y));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
            }
            const int64_t orow = rb * Rb + rp;
            if (lane == 0 && orow < a.rows)
                a.out[int64_t(slot) + (a.out_row0 + orow) * a.ld_out] = c_scale(acc, a.scale);
        }
    }
}

// N == 1: the transform is the identity; only the epilogue (twiddle/select) runs.
template <bool INV>
__global__ void fft_len1_kernel(const FftPassArgs a) {
    const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= a.rows) return;
    FftCta<1, 1, INV> cta{a, nullptr, 0, 0, 1, row, int64_t(blockIdx.y), true};
    cta.gstore(0, cta.gload(0));
}

// O(N^2) direct DFT (any N <= 4096): one thread per (row, frequency).
template <bool INV>
__global__ void dft_direct_kernel(const FftPassArgs a) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = blockIdx.z;
    if (f >= a.N) return;
    FftCta<1, 1, INV> cta{a, nullptr, 0, 0, 1, row, int64_t(blockIdx.y), true};
    double2 acc = make_double2(0.0, 0.0);
    int64_t q = 0;
    for (int k = 0; k < a.N; ++k) {
        acc = c_add(acc, c_mul(cta.gload(k), tw_at(a.tw, q, INV)));
        q += f;
        if (q >= a.N) q -= a.N;
    }
    cta.gstore(f, acc);
}

template <int Rb, int E>
void launch_typed(const FftPassArgs& a, cudaStream_t stream) {
    const int threads = Rb * a.N / E;
    if (threads > 512) throw Error(MNB_ERR_INTERNAL, "fft: more than 512 threads per CTA");
    const size_t smem = size_t(Rb) * a.N * sizeof(double2);
    if (a.blocked) {
        if constexpr (Rb == 8 && E == 16) {
            if (a.N == 1024 && !a.inverse && a.nradix == 3 && a.radix[0] == 16 && a.radix[1] == 16 && a.radix[2] == 4) {
                const size_t sm1024 = size_t(1024) * (8 + 4 + 1 + 1) * sizeof(double2) + 16;
                auto kern = a.mode == FFT_OUT_SELECT ? fft1024_tile_kernel<true> : fft1024_tile_kernel<false>;
                MNB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm1024)));
                const int64_t units = int64_t(ceil_div(a.rows, Rb)) * a.batches;
                const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, a.num_sms)));
                kern<<<grid, 512, sm1024, stream>>>(a);
                MNB_LAUNCH_CHECK();
                return;
            }
        }
        if constexpr (Rb == 8) if (size_t(a.N) * 12 * 16 + 16 <= size_t(227 * 1024)) {
            auto kern = a.inverse ? fft_tile_kernel<E, true> : fft_tile_kernel<E, false>;
            const size_t sm_total = size_t(a.N) * 12 * sizeof(double2) + 16;  // tile + half exchange + barrier
            MNB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_total)));
            const int64_t units = int64_t(ceil_div(a.rows, Rb)) * a.batches;
            // several CTAs per SM for short transforms (registers: <= 128 per thread)
            const int per_sm = int(std::max<size_t>(1, std::min<size_t>({(228 * 1024) / (sm_total + 1024),
                                                                        size_t(2048 / threads),
                                                                        size_t(65536 / (threads * 128))})));
            const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, int64_t(a.num_sms) * per_sm)));
            kern<<<grid, threads, sm_total, stream>>>(a);
            MNB_LAUNCH_CHECK();
            return;
        }
        // otherwise: the generic kernel below, addressing the blocked layout (half or quarter 8-row blocks)
    }
    dim3 grid(ceil_div(a.rows, Rb), unsigned(a.batches));
    auto kern = a.inverse ? fft_pass_kernel<Rb, E, true> : fft_pass_kernel<Rb, E, false>;
    MNB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<grid, threads, smem, stream>>>(a);
    MNB_LAUNCH_CHECK();
}

template <int Rb>
void launch_rb(const FftPassArgs& a, cudaStream_t stream) {
    switch (a.E) {
        case 2: launch_typed<Rb, 2>(a, stream); break;
        case 3: launch_typed<Rb, 3>(a, stream); break;
        case 4: launch_typed<Rb, 4>(a, stream); break;
        case 6: launch_typed<Rb, 6>(a, stream); break;
        case 8: launch_typed<Rb, 8>(a, stream); break;
        case 12: launch_typed<Rb, 12>(a, stream); break;
        case 16: launch_typed<Rb, 16>(a, stream); break;
        case 24: launch_typed<Rb, 24>(a, stream); break;
        default: throw Error(MNB_ERR_INTERNAL, "fft: unsupported elements-per-thread");
    }
}

}  // namespace

bool launch_fft_select_pruned(const FftPassArgs& a, const int32_t* off, const int32_t* ent, int num_sms,
                              cudaStream_t stream) {
    if (a.inverse || a.N % 16 != 0 || a.N / 16 > 128) return false;
    const int U = a.N / 16;
    int Rb = 8;
    while (Rb > 1 && Rb * U > 512) Rb >>= 1;
    const size_t smem = (size_t(a.N) + size_t(Rb) * 16 * U) * sizeof(double2);
    if (smem > size_t(227 * 1024)) return false;
    MNB_CUDA(cudaFuncSetAttribute(fft_select_pruned_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int64_t units = int64_t(ceil_div(a.rows, Rb)) * a.batches;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, num_sms)));
    fft_select_pruned_kernel<<<grid, Rb * U, smem, stream>>>(a, off, ent, Rb, U);
    MNB_LAUNCH_CHECK();
    return true;
}

void launch_fft1024_select(const FftPassArgs& a, const int32_t* off, const int32_t* ent, cudaStream_t stream) {
    const size_t smem = (size_t(1024) * (8 + 1) + 16 * kSB * 8) * sizeof(double2) + (2 * kEnt + 20) * 4 + 16;
    MNB_CUDA(cudaFuncSetAttribute(fft1024_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int64_t units = int64_t(ceil_div(a.rows, 8)) * a.batches;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, a.num_sms)));
    fft1024_select_kernel<<<grid, 512, smem, stream>>>(a, off, ent);
    MNB_LAUNCH_CHECK();
}

bool plan_radices(int N, int& E, int* radix, int& nradix) {
    int m = N, p2 = 0, p3 = 0;
    while (m % 2 == 0) { m /= 2; ++p2; }
    while (m % 3 == 0) { m /= 3; ++p3; }
    if (m != 1) return false;
    nradix = 0;
    if (N == 1) { E = 1; return true; }
    if (p3 == 0) E = N >= 16 ? 16 : N;
    else if (p2 >= 3) E = 24;
    else if (p2 == 2) E = 12;
    else if (p2 == 1) E = 6;
    else E = 3;
    int rem = N;
    const int cand[5] = {16, 8, 4, 3, 2};
    while (rem > 1) {
        int pick = 0;
        for (int R : cand)
            if (E % R == 0 && rem % R == 0) { pick = R; break; }
        if (!pick || nradix >= 10) return false;
        radix[nradix++] = pick;
        rem /= pick;
    }
    return true;
}

void launch_fft_pass(const FftPassArgs& a, cudaStream_t stream) {
    if (a.rows <= 0 || a.batches <= 0) return;
    if (a.N == 1) {
        dim3 grid(ceil_div(a.rows, 128), unsigned(a.batches));
        if (a.inverse) fft_len1_kernel<true><<<grid, 128, 0, stream>>>(a);
        else fft_len1_kernel<false><<<grid, 128, 0, stream>>>(a);
        MNB_LAUNCH_CHECK();
        return;
    }
    switch (a.Rb) {
        case 1: launch_rb<1>(a, stream); break;
        case 2: launch_rb<2>(a, stream); break;
        case 4: launch_rb<4>(a, stream); break;
        case 8: launch_rb<8>(a, stream); break;
        default: throw Error(MNB_ERR_INTERNAL, "fft: unsupported rows per CTA");
    }
}

void launch_dft_direct(const FftPassArgs& a, cudaStream_t stream) {
    if (a.rows <= 0) return;
    require(a.rows <= 65535, MNB_ERR_UNSUPPORTED, "direct DFT: too many rows");
    dim3 grid(ceil_div(a.N, 128), unsigned(a.batches), unsigned(a.rows));
    if (a.inverse) dft_direct_kernel<true><<<grid, 128, 0, stream>>>(a);
    else dft_direct_kernel<false><<<grid, 128, 0, stream>>>(a);
    MNB_LAUNCH_CHECK();
}

}  // namespace mnb

namespace mnb {

namespace {

// Pruned pass B over the blocked layout written by the fused H stage + pass A
// (k_p2fa.cu) for long pass-B lengths, N = 16 U (n = 3 * 2^20: N = 3072, U = 192):
// unit (8-row block, f2, half) reads rows 4 half .. 4 half + 3 of the block's
// [k1][8] column for this f2 (the two halves of a block run on neighbouring CTAs
// at the same time and share every 128-byte line through L2), forms
//   Y_u[j] = sum_q x[u + U q] w_16^{j q}        (u < U, j < 16)
// in registers, and takes each kept frequency as the U-term warp sum
//   X[f1] = sum_u w_N^{f1 u} Y_u[f1 mod 16]
// (the 1024-point version, fft1024_select_kernel, keeps whole tiles in shared memory).
// w_N^k = hi[k >> 6] lo[k & 63] from two small tables.
constexpr int kBEnt = 512;  // staged (f1, slot) pairs per unit

// R rows per unit (R | 8): unit = (8-row block, f2, part), part = which R rows of the block.
// R = 4 (default): 192 KiB of Y in shared memory, one CTA per SM.  R = 2 halves the unit so two
// CTAs share an SM (one's transform and sums over the other's loads); measured slower at c5
// (274 vs 195 ms for both sketches: the per-pair twiddle setup and the ENT staging double).
template <int U, int R>
__global__ void __launch_bounds__(R * U, 4 / R) fft_select_blocked_kernel(const FftPassArgs a,
                                                                          const int32_t* __restrict__ off,
                                                                          const int32_t* __restrict__ ent) {
    constexpr int N = 16 * U, T = R * U, NH = (N + 63) / 64, P = 8 / R;
    extern __shared__ __align__(16) double2 smb[];
    double2* X = smb;                 // Y as [16 j][U u][R r], r slot xor-swizzled by u
    double2* LO = X + 16 * U * R;     // w_N^k, k < 64 (slot-swizzled)
    double2* HI = LO + 64;            // w_N^{64 k}
    int32_t* ENT = reinterpret_cast<int32_t*>(HI + NH);
    const int r = int(threadIdx.x) % R, u = int(threadIdx.x) / R;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31), nwarps = T / 32;
    auto swz = [](int k) { return (k & ~7) | ((k ^ (k >> 3)) & 7); };
    // bank spread of the sums' reads (lanes = consecutive uu): 8 distinct 16-byte groups per phase
    auto xb = [](int j, int uu, int rr) {
        return R == 4 ? (j * U + uu) * 4 + (rr ^ ((uu >> 1) & 3)) : (j * U + uu) * R + (rr ^ ((uu >> 2) & (R - 1)));
    };
    for (int i = threadIdx.x; i < 64; i += T) LO[swz(i)] = __ldg(a.tw + i);
    for (int i = threadIdx.x; i < NH; i += T) HI[i] = __ldg(a.tw + 64 * i);
    const int64_t nrb8 = (a.rows + 7) / 8;
    const int64_t units = nrb8 * a.batches * P;
    const int64_t n1 = N;
    auto load = [&](int64_t unit, double2 (&v)[16]) {
        const int64_t part = unit % P, ub = unit / P;
        const int64_t rb = ub / a.batches, b = ub - rb * a.batches;
        const double2* base = a.in + ((rb * a.batches + b) * n1) * 8 + R * part + r;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const double2* p = base + int64_t(u + U * q) * 8;
            double2 x;
            asm volatile("ld.global.nc.L2::128B.v2.f64 {%0, %1}, [%2];" : "=d"(x.x), "=d"(x.y) : "l"(p));
            v[q] = x;
        }
    };
    double2 v[16];
    int64_t unit = blockIdx.x;
    if (unit < units) load(unit, v);
    for (; unit < units; unit += gridDim.x) {
        const int64_t part = unit % P, ub = unit / P;
        const int64_t rb = ub / a.batches, b = ub - rb * a.batches;
        const int e0 = __ldg(off + b), cnt = __ldg(off + b + 1) - e0;
        dft16_np<false>(v);
        __syncthreads();  // the previous unit's sums are done with X / ENT (and the tables are loaded)
#pragma unroll
        for (int j = 0; j < 16; ++j) X[xb(j, u, r)] = v[d16(j)];
        for (int t = threadIdx.x; t < 2 * min(cnt, kBEnt); t += T) ENT[t] = __ldg(ent + 2 * e0 + t);
        __syncthreads();
        const int64_t next = unit + gridDim.x;
        if (next < units) load(next, v);  // in flight during the sums
        const int32_t* E = cnt <= kBEnt ? ENT : ent + 2 * e0;
        for (int p0 = warp; p0 < R * cnt; p0 += 2 * nwarps) {
            double vv[4];
            int slot2[2], row2[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int p = p0 + nwarps * k;
                const bool ok = p < R * cnt;
                const int rp = p % R, s = ok ? p / R : 0;
                const int f = E[2 * s];
                slot2[k] = ok ? E[2 * s + 1] : -1;
                row2[k] = rp;
                const int j = f & 15;
                double2 acc = make_double2(0.0, 0.0);
                // w^{f uu}, uu = lane + 32 t: w^{f lane} times (w^{32 f})^t
                const int k0 = int((int64_t(f) * lane) % N), ks = int((int64_t(f) * 32) % N);
                double2 w = c_mul(HI[k0 >> 6], LO[swz(k0 & 63)]);
                const double2 wstep = c_mul(HI[ks >> 6], LO[swz(ks & 63)]);
#pragma unroll
                for (int t = 0; t < (U + 31) / 32; ++t) {
                    const int uu = lane + 32 * t;
                    if (uu < U) {
                        const double2 y = X[xb(j, uu, rp)];
                        acc.x = fma(y.x, w.x, fma(-y.y, w.y, acc.x));
                        acc.y = fma(y.x, w.y, fma(y.y, w.x, acc.y));
                    }
                    w = c_mul(w, wstep);
                }
                vv[2 * k] = acc.x;
                vv[2 * k + 1] = acc.y;
            }
            xreduce4(vv, lane);
            const double other = __shfl_down_sync(0xffffffffu, vv[0], 8);
            if ((lane & 15) == 0) {
                const int k = lane >> 4;
                const int64_t row = rb * 8 + R * part + row2[k];
                if (slot2[k] >= 0 && row < a.rows)
                    a.out[int64_t(slot2[k]) + (a.out_row0 + row) * a.ld_out] = c_scale(make_double2(vv[0], other), a.scale);
            }
        }
    }
}

// Radix-8 variant for N = 8 U (n = 3 * 2^20: U = 384), 2 rows per unit, 768 threads: each thread
// holds only 8 values (32 registers), so the transform and the prefetched next unit fit in the 80
// registers a 768-thread CTA gets -- the radix-16 kernel above spills there (its 16 complex values
// alone take 64 registers), and the spills clog the load pipe (lg_throttle 45 % of its stalls).
//   Y_u[j] = sum_q x[u + U q] w_8^{j q}  (q, j < 8),   X[f] = sum_{u < U} w_N^{f u} Y_u[f mod 8]
template <int U>
__global__ void __launch_bounds__(2 * U, 1) fft_select_blocked8_kernel(const FftPassArgs a,
                                                                      const int32_t* __restrict__ off,
                                                                      const int32_t* __restrict__ ent) {
    constexpr int R = 2, N = 8 * U, T = R * U, NH = (N + 63) / 64, P = 8 / R;
    extern __shared__ __align__(16) double2 smb[];
    double2* X = smb;                 // Y as [8 j][U u][2 r], r slot xor-swizzled by u
    double2* LO = X + 8 * U * R;      // w_N^k, k < 64 (slot-swizzled)
    double2* HI = LO + 64;            // w_N^{64 k}
    int32_t* ENT = reinterpret_cast<int32_t*>(HI + NH);
    const int r = int(threadIdx.x) % R, u = int(threadIdx.x) / R;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31), nwarps = T / 32;
    auto swz = [](int k) { return (k & ~7) | ((k ^ (k >> 3)) & 7); };
    auto xb = [](int j, int uu, int rr) { return (j * U + uu) * R + (rr ^ ((uu >> 2) & 1)); };
    for (int i = threadIdx.x; i < 64; i += T) LO[swz(i)] = __ldg(a.tw + i);
    for (int i = threadIdx.x; i < NH; i += T) HI[i] = __ldg(a.tw + 64 * i);
    const int64_t nrb8 = (a.rows + 7) / 8;
    const int64_t units = nrb8 * a.batches * P;
    auto load = [&](int64_t unit, double2 (&v)[8]) {
        const int64_t part = unit % P, ub = unit / P;
        const int64_t rb = ub / a.batches, b = ub - rb * a.batches;
        const double2* base = a.in + ((rb * a.batches + b) * int64_t(N)) * 8 + R * part + r;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double2* p = base + int64_t(u + U * q) * 8;
            double2 x;
            asm volatile("ld.global.nc.L2::128B.v2.f64 {%0, %1}, [%2];" : "=d"(x.x), "=d"(x.y) : "l"(p));
            v[q] = x;
        }
    };
    double2 v[8];
    int64_t unit = blockIdx.x;
    if (unit < units) load(unit, v);
    for (; unit < units; unit += gridDim.x) {
        const int64_t part = unit % P, ub = unit / P;
        const int64_t rb = ub / a.batches, b = ub - rb * a.batches;
        const int e0 = __ldg(off + b), cnt = __ldg(off + b + 1) - e0;
        dft8<false>(v);
        __syncthreads();  // the previous unit's sums are done with X / ENT (and the tables are loaded)
#pragma unroll
        for (int j = 0; j < 8; ++j) X[xb(j, u, r)] = v[j];
        for (int t = threadIdx.x; t < 2 * min(cnt, kBEnt); t += T) ENT[t] = __ldg(ent + 2 * e0 + t);
        __syncthreads();
        const int64_t next = unit + gridDim.x;
        if (next < units) load(next, v);  // in flight during the sums
        const int32_t* E = cnt <= kBEnt ? ENT : ent + 2 * e0;
        for (int p0 = warp; p0 < R * cnt; p0 += 2 * nwarps) {
            double vv[4];
            int slot2[2], row2[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int p = p0 + nwarps * k;
                const bool ok = p < R * cnt;
                const int rp = p % R, s = ok ? p / R : 0;
                const int f = E[2 * s];
                slot2[k] = ok ? E[2 * s + 1] : -1;
                row2[k] = rp;
                const int j = f & 7;
                double2 acc = make_double2(0.0, 0.0);
                // w^{f uu}, uu = lane + 32 t: w^{f lane} times (w^{32 f})^t  (f lane < 2^17: 32-bit)
                const int k0 = (f * lane) % N, ks = (f * 32) % N;
                double2 w = c_mul(HI[k0 >> 6], LO[swz(k0 & 63)]);
                const double2 wstep = c_mul(HI[ks >> 6], LO[swz(ks & 63)]);
#pragma unroll
                for (int t = 0; t < U / 32; ++t) {
                    const double2 y = X[xb(j, lane + 32 * t, rp)];
                    acc.x = fma(y.x, w.x, fma(-y.y, w.y, acc.x));
                    acc.y = fma(y.x, w.y, fma(y.y, w.x, acc.y));
                    w = c_mul(w, wstep);
                }
                vv[2 * k] = acc.x;
                vv[2 * k + 1] = acc.y;
            }
            xreduce4(vv, lane);
            const double other = __shfl_down_sync(0xffffffffu, vv[0], 8);
            if ((lane & 15) == 0) {
                const int k = lane >> 4;
                const int64_t row = rb * 8 + R * part + row2[k];
                if (slot2[k] >= 0 && row < a.rows)
                    a.out[int64_t(slot2[k]) + (a.out_row0 + row) * a.ld_out] = c_scale(make_double2(vv[0], other), a.scale);
            }
        }
    }
}

// Pass B for SHORT second passes (N = 128 ... 512: n = N x 1024, BASELINE c3 is 128 x 1024), pruned to
// the sampled frequencies and taken directly: with l / 1024 (a handful of) kept outputs per f2, the
// N-term sums X[f1] = sum_k1 Y[k1] w_N^{f1 k1} cost less than any transform of the unit, and the
// kernel is a pure stream over pass A's blocked output [row block][f2][k1][8 rows] (16 KiB units at
// N = 128).  Thread (r, q): row r of the block, k1 = q + 32 j (j < NJ = N / 32) -- a warp reads 512
// contiguous bytes per j; the next unit's values are in flight during the sums.  Per kept output the
// 32 q-partials of a row meet by two shuffles (the 4 q of a warp) and a fixed-order sum over the 8
// warps through shared memory (one barrier per unit, 16 outputs at a time).
template <int NJ>
__global__ void __launch_bounds__(256, (NJ <= 4 ? 4 : NJ <= 8 ? 2 : 1)) fft_select_blocked_direct_kernel(const FftPassArgs a,
                                                                           const int32_t* __restrict__ off,
                                                                           const int32_t* __restrict__ ent) {
    constexpr int N = 32 * NJ, T = 256, EB = 16;
    extern __shared__ int32_t OFF[];     // the CSR offsets of every f2 (batches + 1)
    __shared__ double2 TW[N];
    __shared__ double2 part[EB][8][8];   // [entry][warp][row]
    __shared__ int32_t ENT[2][2 * EB];   // double-buffered (f1, slot) pairs of the current chunk
    const int r = int(threadIdx.x) & 7, q = int(threadIdx.x) >> 3;
    const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
    for (int i = threadIdx.x; i < N; i += T) TW[i] = __ldg(a.tw + i);
    for (int i = threadIdx.x; i <= a.batches; i += T) OFF[i] = __ldg(off + i);
    __syncthreads();
    const int64_t nrb8 = (a.rows + 7) / 8;
    const int64_t units = nrb8 * a.batches;
    auto load = [&](int64_t unit, double2 (&v)[NJ]) {
        const double2* base = a.in + unit * int64_t(N) * 8 + r;  // unit = rb * batches + b
#pragma unroll
        for (int j = 0; j < NJ; ++j) v[j] = __ldg(base + int64_t(q + 32 * j) * 8);
    };
    // this thread's word of a unit's first chunk of entries (threads < 2 EB), fetched a unit ahead
    auto first_entries = [&](int64_t unit) -> int32_t {
        const int b = int(unit % a.batches);
        const int e0 = OFF[b], cnt = OFF[b + 1] - e0;
        return int(threadIdx.x) < 2 * min(cnt, EB) ? __ldg(ent + 2 * e0 + threadIdx.x) : 0;
    };
    double2 v[NJ], vn[NJ];
    int32_t my_ent = 0, my_ent_n = 0;
    int64_t unit = blockIdx.x;
    if (unit < units) {
        load(unit, v);
        my_ent = first_entries(unit);
    }
    int buf = 0;
    for (; unit < units; unit += gridDim.x) {
        const int64_t rb = unit / a.batches, b = unit - rb * a.batches;
        const int e0 = OFF[b], cnt = OFF[b + 1] - e0;
        const int64_t next = unit + gridDim.x;
        if (next < units) {
            load(next, vn);
            my_ent_n = first_entries(next);
        }
        for (int c0 = 0; c0 < cnt; c0 += EB) {
            const int nc = min(EB, cnt - c0);
            if (int(threadIdx.x) < 2 * nc)
                ENT[buf][threadIdx.x] = c0 == 0 ? my_ent : __ldg(ent + 2 * (e0 + c0) + threadIdx.x);
            __syncthreads();  // entries staged; the previous chunk's partials have been read
            for (int e = 0; e < nc; ++e) {
                const int f = ENT[buf][2 * e];
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const double2 w = TW[(f * (q + 32 * j)) & (N - 1)];
                    acc.x = fma(v[j].x, w.x, fma(-v[j].y, w.y, acc.x));
                    acc.y = fma(v[j].x, w.y, fma(v[j].y, w.x, acc.y));
                }
                // the warp's 4 values of q (lanes r, r + 8, r + 16, r + 24)
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 8);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 8);
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
                if (lane < 8) part[e][warp][lane] = acc;
            }
            __syncthreads();
            if (int(threadIdx.x) < 8 * nc) {
                const int e = int(threadIdx.x) >> 3, rr = int(threadIdx.x) & 7;
                double2 sum = part[e][0][rr];
#pragma unroll
                for (int w = 1; w < 8; ++w) {
                    sum.x += part[e][w][rr].x;
                    sum.y += part[e][w][rr].y;
                }
                const int64_t row = rb * 8 + rr;
                if (row < a.rows)
                    a.out[int64_t(ENT[buf][2 * e + 1]) + (a.out_row0 + row) * a.ld_out] = c_scale(sum, a.scale);
            }
            buf ^= 1;  // the writers above still read this buffer while the next chunk is staged
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) v[j] = vn[j];
        my_ent = my_ent_n;
    }
}

template <int NJ>
void launch_direct(const FftPassArgs& a, const int32_t* off, const int32_t* ent, int num_sms, cudaStream_t stream) {
    const int64_t units = int64_t(ceil_div(a.rows, 8)) * a.batches;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, int64_t(num_sms) * (NJ <= 4 ? 4 : NJ <= 8 ? 2 : 1))));
    fft_select_blocked_direct_kernel<NJ><<<grid, 256, size_t(a.batches + 1) * 4, stream>>>(a, off, ent);
    MNB_LAUNCH_CHECK();
}

}  // namespace

bool launch_fft_select_blocked(const FftPassArgs& a, const int32_t* off, const int32_t* ent, int num_sms,
                               cudaStream_t stream) {
    if (!a.inverse && (a.N == 128 || a.N == 256 || a.N == 512)) {
        if (a.N == 128) launch_direct<4>(a, off, ent, num_sms, stream);
        else if (a.N == 256) launch_direct<8>(a, off, ent, num_sms, stream);
        else launch_direct<16>(a, off, ent, num_sms, stream);
        return true;
    }
    if (a.inverse || a.N != 3072) return false;
    static const int radix = [] { const char* e = std::getenv("MNB_FB_RADIX"); return e && std::atoi(e) == 16 ? 16 : 8; }();
    if (radix == 8) {
        constexpr int U8 = 384;
        const size_t smem = (size_t(8) * U8 * 2 + 64 + (a.N + 63) / 64) * sizeof(double2) + 2 * kBEnt * 4;
        auto k = fft_select_blocked8_kernel<U8>;
        MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const int64_t units = int64_t(ceil_div(a.rows, 8)) * a.batches * 4;
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, num_sms)));
        k<<<grid, 2 * U8, smem, stream>>>(a, off, ent);
        MNB_LAUNCH_CHECK();
        return true;
    }
    constexpr int U = 192;
    // 4-row units, one CTA per SM (2-row units on two CTAs per SM measured slower: 274 vs 195 ms
    // for both c5 sketches; MNB_FB_ROWS=2 selects them)
    static const int R = [] { const char* e = std::getenv("MNB_FB_ROWS"); return e && std::atoi(e) == 2 ? 2 : 4; }();
    const size_t smem = (size_t(16) * U * R + 64 + (a.N + 63) / 64) * sizeof(double2) + 2 * kBEnt * 4;
    const int64_t units = int64_t(ceil_div(a.rows, 8)) * a.batches * (8 / R);
    const int per_sm = R == 2 ? 2 : 1;  // resident CTAs per SM (shared memory: 2 x 101 KiB or 1 x 197 KiB)
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, int64_t(num_sms) * per_sm)));
    if (R == 4) {
        auto k = fft_select_blocked_kernel<U, 4>;
        MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k<<<grid, 4 * U, smem, stream>>>(a, off, ent);
    } else {
        auto k = fft_select_blocked_kernel<U, 2>;
        MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k<<<grid, 2 * U, smem, stream>>>(a, off, ent);
    }
    MNB_LAUNCH_CHECK();
    return true;
}

}  // namespace mnb
