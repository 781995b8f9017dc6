// Sketch H stage, forward chain, for row blocks of the problem matrix
// (src/srft.cpp:49-58 applied by apply_to_columns, src/srft.cpp:147-153).
//
// Same arithmetic as k_hstage.cu (bit-identical results), restructured for
// bandwidth: the old kernel waited on a dependent index load and then a
// data load every 8 steps (latency-bound, ~2.4 TB/s).  Here
//   * one persistent CTA per SM walks work items (row block x chunk);
//   * per item, thread 0 bulk-copies the chunk's gather indices and its
//     per-step parameter records {cs_j, zin_j, zout_{j+1}} (48 B, built once
//     per operator by build_chain_params) into shared memory;
//   * every thread owns one row and streams its gathered elements through a
//     private (D+1)-slot cp.async ring D steps ahead of the scan, so each SM
//     keeps ~D * 2 KiB of reads in flight with no cross-thread barrier;
//   * outputs are stored straight from registers (a warp writes 32
//     consecutive rows = 512 contiguous bytes per index).
//
// Scan (rotation_chain_scalar, src/kernels_scalar.cpp:15-24), per chunk
// [i0, i1) restarted at the host halo start `start` (host_srft.cpp):
//   carry = x_start;  for j = start-1 .. lo:  carry' = c x_j + s carry,
//   out[j+1] = -s x_j + c carry  (if j+1 < i1);   out[0] = carry (chunk 0).
#include "common.cuh"
#include "kernels.cuh"

namespace mnb {

namespace {

constexpr int kRows = 128;  // rows (threads) per CTA

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct ChainSmem {
    size_t ring, params, idx, bar, total;
};
__host__ __device__ inline ChainSmem chain_smem(int D, int esz, int64_t max_span) {
    ChainSmem L;
    L.ring = 0;
    L.params = (size_t(D + 1) * kRows * esz + 127) & ~size_t(127);
    L.idx = L.params + ((size_t(max_span) * 48 + 127) & ~size_t(127));
    L.bar = L.idx + ((size_t(max_span + 8) * 4 + 127) & ~size_t(127));
    L.total = L.bar + 16;
    return L;
}

// FIRST: the first H half (conj input, zin, finiteness check); else the second.
template <bool REAL, bool FIRST, int D>
__global__ void __launch_bounds__(kRows, 2) hchain_kernel(const HChainArgs a) {
    using ET = typename std::conditional<REAL, double, double2>::type;
    constexpr int esz = int(sizeof(ET));
    extern __shared__ __align__(128) unsigned char smem[];
    const ChainSmem L = chain_smem(D, esz, a.max_span);
    ET* ring = reinterpret_cast<ET*>(smem + L.ring) + threadIdx.x;  // this thread's column of the ring
    const double2* prm = reinterpret_cast<const double2*>(smem + L.params);
    const int32_t* gix = reinterpret_cast<const int32_t*>(smem + L.idx);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
    const int r = threadIdx.x;
    if (r == 0) {
        mbar_init1(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int64_t nrb = (a.rows + kRows - 1) / kRows;
    const int64_t items = nrb * a.nchunks;
    const ET* in = static_cast<const ET*>(a.in);
    const int64_t ld_in = a.ld_in, ld_out = a.ld_out;
    uint32_t phase = 0;
    bool bad = false;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t c = item / nrb, rb = item - c * nrb;
        const int64_t i0 = c * a.chunk, i1 = min(a.n, i0 + a.chunk);
        const int64_t start = __ldg(a.halo + c);
        const int64_t lo = i0 > 0 ? i0 - 1 : 0;
        const int Q = int(start - lo + 1);
        const int64_t lo4 = lo & ~int64_t(3);           // 16-byte aligned index window
        const int64_t hi4 = (start + 4) & ~int64_t(3);  // <= n+3: inside the 256-byte padded parameter blob
        if (r == 0) {
            const uint32_t pbytes = uint32_t(Q) * 48, ibytes = uint32_t(hi4 - lo4) * 4;
            mbar_expect(bar, pbytes + ibytes);
            bulk_copy(smem + L.params, a.params + 3 * lo, pbytes, bar);
            bulk_copy(smem + L.idx, a.gather + lo4, ibytes, bar);
        }
        mbar_wait_parity(bar, phase);
        phase ^= 1u;

        const int64_t row = rb * kRows + r;
        const bool live = row < a.rows;
        const ET* src = in + (a.in_row0 + (live ? row : 0));
        // entry e (ascending j = lo + e); step q walks e = Q-1 .. 0
        const int32_t* G = gix + (lo - lo4);
#pragma unroll 1
        for (int q = 0; q < D; ++q) {
            if (q < Q) cp_async<esz>(ring + q * kRows, src + int64_t(G[Q - 1 - q]) * ld_in);
            cp_commit();
        }
        int e = Q - 1;      // entry of the step being consumed
        int slot = 0;       // ring slot of that step
        auto fetch = [&]() -> double2 {
            cp_wait<D - 1>();
            const ET v = ring[slot * kRows];
            // refill: entry e - D into the slot consumed one step ago
            int sn = slot == 0 ? D : slot - 1;
            if (e - D >= 0) cp_async<esz>(ring + sn * kRows, src + int64_t(G[e - D]) * ld_in);
            cp_commit();
            slot = slot == D ? 0 : slot + 1;
            double2 x;
            if constexpr (REAL) x = make_double2(v, 0.0);
            else x = v;
            if constexpr (FIRST) {
                bad |= !(isfinite(x.x) && isfinite(x.y));
                x.y = -x.y;                         // column of B = A^H is conj(row of A)
                x = c_mul_rn(x, prm[3 * e + 1]);    // Z~ at the gathered index
            }
            return x;
        };
        double2 carry = fetch();  // x_start
        --e;
        // halo steps (outputs at j+1 >= i1 are another chunk's) then the chunk's own steps
        const int e_store = int(i1 - 1 - lo);  // j + 1 < i1  <=>  e < e_store
        // output pointer of index o = lo + e + 1, walked downwards one index per step
        const bool blk = a.blk_n1 > 0;
        const int64_t n1 = a.blk_n1, n2 = a.blk_n2;
        double2* obase = blk ? a.out + (row >> 3) * a.n * 8 + (row & 7) : a.out + (a.out_row0 + row);
        int64_t k1 = 0;
        double2* optr;
        if (blk) {
            const int64_t o = lo + e + 1;
            k1 = o % n1;
            optr = obase + (k1 * n2 + o / n1) * 8;
        } else {
            optr = obase + (lo + e + 1) * ld_out;
        }
        const int64_t wrap = ((n1 - 1) * n2 - 1) * 8, dstep = blk ? n2 * 8 : ld_out;
        auto step = [&](bool store) {
            const double2 x = fetch();
            const double2 cs = prm[3 * e];
            const double c_ = cs.x, s_ = cs.y;
            const double2 nc = make_double2(__dadd_rn(__dmul_rn(c_, x.x), __dmul_rn(s_, carry.x)),
                                            __dadd_rn(__dmul_rn(c_, x.y), __dmul_rn(s_, carry.y)));
            if (store) {
                double2 o = make_double2(__dadd_rn(__dmul_rn(-s_, x.x), __dmul_rn(c_, carry.x)),
                                         __dadd_rn(__dmul_rn(-s_, x.y), __dmul_rn(c_, carry.y)));
                o = c_mul_rn(o, prm[3 * e + 2]);    // output diagonal at j + 1
                if (live) *optr = o;
            }
            carry = nc;
            if (blk && k1 == 0) {
                k1 = n1 - 1;
                optr += wrap;
            } else {
                --k1;
                optr -= dstep;
            }
            --e;
        };
#pragma unroll 1
        while (e >= e_store) step(false);
#pragma unroll 2
        while (e >= 0) step(true);
        if (i0 == 0 && live) *obase = c_mul_rn(carry, a.zout0);
        cp_wait_all();
        __syncthreads();  // the parameter window is reused by the next item
    }
    if constexpr (FIRST)
        if (bad && a.nonfinite) *a.nonfinite = 1;
}

// rec[j] = {cs_j, zin_j, zout_{j+1}}  (zout_n = 1)
__global__ void build_chain_params_kernel(const double2* __restrict__ cssn, const double2* __restrict__ zin,
                                          const int32_t* __restrict__ zin_index, const double2* __restrict__ zout,
                                          int64_t n, double2* __restrict__ rec) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    rec[3 * j] = cssn[j];
    rec[3 * j + 1] = zin ? zin[zin_index ? zin_index[j] : j] : make_double2(1.0, 0.0);
    rec[3 * j + 2] = (zout && j + 1 < n) ? zout[j + 1] : make_double2(1.0, 0.0);
}

template <bool REAL, bool FIRST, int D>
void launch_typed(const HChainArgs& a, int num_sms, cudaStream_t stream) {
    const ChainSmem L = chain_smem(D, REAL ? 8 : 16, a.max_span);
    auto k = hchain_kernel<REAL, FIRST, D>;
    MNB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total)));
    const int64_t items = ((a.rows + kRows - 1) / kRows) * a.nchunks;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(items, 2 * num_sms)));
    k<<<grid, kRows, L.total, stream>>>(a);
    MNB_LAUNCH_CHECK();
}

}  // namespace

bool hchain_fits(int64_t max_span, int is_real) {
    return chain_smem(16, is_real ? 8 : 16, max_span).total <= size_t(227 * 1024);
}

// Two CTAs per SM when the ring (D = 24) and the parameter window fit in half
// the shared memory; otherwise one CTA with a deeper ring.
void launch_hchain(const HChainArgs& a, int num_sms, cudaStream_t stream) {
    if (a.rows <= 0) return;
    const int esz = a.in_real ? 8 : 16;
    const bool first = a.has_zin != 0;
    const bool two = chain_smem(24, esz, a.max_span).total <= size_t(113 * 1024);
#define MNB_HCHAIN(R, F)                                           \
    do {                                                           \
        if (two) launch_typed<R, F, 24>(a, num_sms, stream);       \
        else launch_typed<R, F, 16>(a, num_sms, stream);           \
    } while (0)
    if (a.in_real) {
        if (first) MNB_HCHAIN(true, true);
        else MNB_HCHAIN(true, false);
    } else {
        if (first) MNB_HCHAIN(false, true);
        else MNB_HCHAIN(false, false);
    }
#undef MNB_HCHAIN
}

void build_chain_params(const double2* cssn, const double2* zin, const int32_t* zin_index, const double2* zout,
                        int64_t n, double2* rec, cudaStream_t stream) {
    build_chain_params_kernel<<<ceil_div(n, 256), 256, 0, stream>>>(cssn, zin, zin_index, zout, n, rec);
    MNB_LAUNCH_CHECK();
}

}  // namespace mnb
