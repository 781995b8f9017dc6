// Fused second H stage + four-step FFT pass A of the sketch (sm_100a), for
// n = n1 x 1024 (n1 = 1024 or 3072) with rotation-chain chunks of n1 indices.
//
// The unfused path runs P2 (x2 = D Chain(x1[:, p_i]), src/srft.cpp:56-57,128)
// and then pass A (length-1024 DFTs over k2 of x2[:, k1 + n1 k2]) as two
// launches with x2 (16 B per element) written to HBM and read back.  But
// chunk c of P2's chain IS k2 = c, and every chunk walks its k1 range in the
// same (descending) order: if all 1024 chunks of a row block advance in
// lock step, step s produces x2[:, k1 + n1 k2] for one k1 = n1 - 1 - s and
// every k2 -- exactly one pass-A transform.  So one CTA (512 threads) owns 4
// rows and all 1024 chunks (a cluster pair covers an 8-row block); each step it
//   1. advances 8 chains per thread (row r, chunks c = u + 128 q) with the
//      gathered x1 values that landed during the previous step (a 64-byte
//      piece of 4 rows per gathered index, the 4 row-lanes of a chunk coalesced;
//      the cluster partner reads the other half of the 128-byte piece),
//   2. transforms the 1024 chain outputs of each row: radix 8 in registers (the
//      chain outputs already sit in its input order), radix 8 and radix 16 through
//      two shared-memory exchanges, the last radix 2 of the radix 16 by shuffles,
//   3. applies the four-step twiddle w_n^{f2 k1} and stores the 1024 results
//      per row in the blocked layout [row block][f2][k1][8] pass B reads.
// x2 never exists in HBM: the sketch reads x1 once and writes pass A's output
// once (2 x 16 B per element instead of 4 x 16 B).  A row block whose 1024 (or
// n1) steps would leave most pairs idle in the last round runs as two k1
// segments, the second restarted like a chunk boundary (restart table of n1/2-
// index sub-chunks).
//
// Chain arithmetic (rotation_chain_scalar, src/kernels_scalar.cpp:15-24) is
// the hchain_kernel's, operation for operation (same _rn intrinsics, same
// restart points), so x2 -- and hence the FFT input -- is bit-identical.
#include "common.cuh"
#include "fft_dev.cuh"
#include "kernels.cuh"

namespace mnb {

namespace {

constexpr int kN = 1024;       // pass-A length n2 = number of chunks
constexpr int kRows = 4;       // rows per CTA; a cluster of 2 CTAs covers one 8-row block
constexpr int kThreads = 512;  // chain phase: (r, u): r = tid & 3, u = tid >> 2 in [0, 128)
constexpr int kQ = 8;          // chunks per thread: c = u + 128 q
constexpr int kPad = 17;       // stage-3 exchange rows padded to 17 entries (bank spread)

// The length-1024 transform over k2 = c of each row, c = u + 128 q, u = u1 + 16 u2:
//   stage 1 (chain threads, radix 8 over q):  Y1[u][a]  = sum_q x[u + 128 q] w_8^{qa} * w_1024^{ua}
//   stage 2 (radix 8 over u2):                Y2[u1][a][b1] = sum_u2 Y1[u1 + 16 u2][a] w_8^{u2 b1} * w_128^{u1 b1}
//   stage 3 (radix 16 over u1):               X[a + 8 b1 + 64 b2] = sum_u1 Y2[u1][a][b1] w_16^{u1 b2}
// (w_1024^{c f} with f = a + 8 (b1 + 8 b2) factors exactly so.)
//
// Shared memory (202 KiB, one CTA per SM):
//   X    exchange buffer: Y1 as [a][u][r] (64 KiB), Y2 as [b1][a][u1 (17)][r] (68 KiB)
//   PRM  [1024][2] double2  this step's chain records {cs_j, d_{j+1}} per chunk
//   IDX  [1024] int32       the next step's gather indices
//   W    [1024] double2     w_1024^k
//   Z    [1024] double2     this step's four-step twiddles w_n^{f k1}
//   L    [8][512] double2   thread-private landing slots of the next step's gathered
//                           values (cp.async, refilled as soon as a value is consumed)
// PRM, IDX and Z come from step-major tables (build_p2fa_tables) with one TMA bulk
// copy each per step, issued by thread 0 a phase ahead of their use.  The two CTAs
// of a cluster own rows 0-3 and 4-7 of one 8-row block and advance in lock step (a
// cluster barrier every 16 steps), so their 64-byte halves of every gathered
// 128-byte piece reach L2 together (the loads ask L2 for the whole line) and the
// blocked stores of the pair fill whole lines.
struct P2faSmem {
    static constexpr size_t X = 0;
    static constexpr size_t PRM = X + size_t(64) * kPad * kRows * 16;
    static constexpr size_t IDX = PRM + size_t(kN) * 32;
    static constexpr size_t W = IDX + size_t(kN) * 4;
    static constexpr size_t Z = W + size_t(kN) * 16;
    static constexpr size_t L = Z + size_t(kN) * 16;
    static constexpr size_t BAR = L + size_t(kQ) * kThreads * 16;
    static constexpr size_t TOTAL = BAR + 16;
};

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(dst)),
                 "l"(src), "r"(bytes), "r"(sa(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(sa(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void cp_pair(void* dst, const void* src) {  // 16 B, L2 fetches the 128-byte line
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(sa(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// gathered 64-byte half-piece: ask L2 for the whole 128-byte line, which the cluster
// partner reads next (read-only for the kernel's lifetime)
__device__ __forceinline__ double2 ld_pair(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L2::128B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1) p2fa_kernel(const P2faArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    double2* X = reinterpret_cast<double2*>(smem + P2faSmem::X);
    double2* PRM = reinterpret_cast<double2*>(smem + P2faSmem::PRM);
    int32_t* IDX = reinterpret_cast<int32_t*>(smem + P2faSmem::IDX);
    double2* Ws = reinterpret_cast<double2*>(smem + P2faSmem::W);
    double2* Zs = reinterpret_cast<double2*>(smem + P2faSmem::Z);
    double2* Lt = reinterpret_cast<double2*>(smem + P2faSmem::L) + threadIdx.x;  // slot q at Lt[q * kThreads]
    uint64_t* barA = reinterpret_cast<uint64_t*>(smem + P2faSmem::BAR);         // PRM(s) + IDX(s+1)
    uint64_t* barZ = barA + 1;                                                   // Z(s)
    const int n1 = a.n1;  // chain chunk = k1 steps per row block (1024 or 3072)
    const int tid = int(threadIdx.x);
    const int r = tid & 3, u = tid >> 2;                        // chain / stage 1
    const int u1 = (tid >> 2) & 15, a8 = tid >> 6;              // stage 2: (r, u1, a)
    const int h3 = (tid >> 2) & 1, a3 = (tid >> 3) & 7, b13 = tid >> 6;  // stage 3: (r, h, a, b1)
    const int rank = int(blockIdx.x & 1);  // cluster rank: rows 4 rank .. 4 rank + 3 of the block
    for (int i = tid; i < kN; i += kThreads) Ws[i] = __ldg(a.tw + i);
    if (tid == 0) {
        mbar_init(barA);
        mbar_init(barZ);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phA = 0, phZ = 0;

    const int64_t nrb = a.rows / 8;
    const int64_t ld = a.ld;
    // step-major tables: step s of chunk c stores j = 1024 c + 1022 - s (out index j + 1);
    // chunk 0's last output (s = 1023, index 0) is the final carry times d_0
    auto stage_a = [&](int sp, int si) {  // PRM(sp) and (si < 1024) IDX(si): thread 0
        fence_async_smem();
        const uint32_t bytes = uint32_t(kN) * 32 + (si < n1 ? uint32_t(kN) * 4 : 0u);
        mbar_expect(barA, bytes);
        bulk_load(PRM, a.rec_t + size_t(sp) * kN * 2, uint32_t(kN) * 32, barA);
        if (si < n1) bulk_load(IDX, a.idx_t + size_t(si) * kN, uint32_t(kN) * 4, barA);
    };
    auto stage_z = [&](int k1) {
        fence_async_smem();
        mbar_expect(barZ, uint32_t(kN) * 16);
        bulk_load(Zs, a.z_t + size_t(k1) * kN, uint32_t(kN) * 16, barZ);
    };

    // (the loop bound is uniform across the cluster: both CTAs run the same row blocks)
    // work units: (row block, k1 segment); segment g covers steps [g S, (g + 1) S), S = n1 / nseg
    // units: row blocks [0, full_rb) whole, the rest as two k1 segments each (restarted from the
    // half-chunk restart table), so the last pair round can be a half round
    const int64_t full = min(a.full_rb, nrb);
    const int64_t units = full + 2 * (nrb - full);
    for (int64_t unit = blockIdx.x >> 1; unit < units; unit += gridDim.x >> 1) {
        int64_t rb;
        int seg, nseg;
        if (unit < full) {
            rb = unit;
            seg = 0;
            nseg = 1;
        } else {
            rb = full + ((unit - full) >> 1);
            seg = int((unit - full) & 1);
            nseg = 2;
        }
        const int S = n1 / nseg;
        const int s0 = seg * S, s1 = s0 + S;
        const double2* src = a.x1 + (rb * 8 + kRows * rank + r);
        double2 carry[kQ];
        // ---- each chunk's carry at the segment's upper bound, from the restart pass
        //      (p2fa_carry_kernel: hchain_kernel's non-storing steps, start-1 .. B-1)
        {
            const int64_t crow = rb * 8 + kRows * rank + r;
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const int c = u + 128 * q;
                carry[q] = a.carries[int64_t(seg == 0 ? c : kN + c) * a.ldc + crow];
            }
        }
        // ---- values(0) straight from the step-0 index row; PRM(0) + IDX(1), Z(0) by TMA
        __syncthreads();  // the previous row block is done with PRM / IDX / Z / X
        if (tid == 0) {
            stage_a(s0, s0 + 1);
            stage_z(n1 - 1 - s0);
        }
#pragma unroll
        for (int q = 0; q < kQ; ++q) cp_pair(Lt + q * kThreads, src + int64_t(__ldg(a.idx_t + size_t(s0) * kN + u + 128 * q)) * ld);
        cp_commit();
        cp_wait_all();
        cluster_sync();

        double2* orow = a.out + rb * int64_t(kN) * n1 * 8 + kRows * rank + r;
#pragma unroll 1
        for (int s = s0; s < s1; ++s) {
            const int k1 = n1 - 1 - s;
            const bool more = s + 1 < s1;
            mbar_wait(barA, phA);  // PRM(s), IDX(s+1)
            phA ^= 1u;
            // 1. chain steps (hchain_kernel's storing step) on values(s); each landing slot is
            //    refilled with values(s+1) as soon as its value has been consumed
            double2 v[16];
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const int c = u + 128 * q;
                const double2 x = Lt[q * kThreads];
                if (c == 0 && s == n1 - 1) {
                    v[q] = c_mul_rn(carry[q], a.zout0);  // out[0] = carry * d_0
                } else {
                    const double2 cs = PRM[2 * c], zo = PRM[2 * c + 1];
                    const double c_ = cs.x, s_ = cs.y;
                    const double2 nc = make_double2(__dadd_rn(__dmul_rn(c_, x.x), __dmul_rn(s_, carry[q].x)),
                                                    __dadd_rn(__dmul_rn(c_, x.y), __dmul_rn(s_, carry[q].y)));
                    const double2 o = make_double2(__dadd_rn(__dmul_rn(-s_, x.x), __dmul_rn(c_, carry[q].x)),
                                                   __dadd_rn(__dmul_rn(-s_, x.y), __dmul_rn(c_, carry[q].y)));
                    v[q] = c_mul_rn(o, zo);
                    carry[q] = nc;
                }
                if (more && !(c == 0 && s + 1 == n1 - 1))
                    cp_pair(Lt + q * kThreads, src + int64_t(IDX[c]) * ld);
            }
            cp_commit();
            // 2. stage 1: radix 8 over q, twiddle w_1024^{u a} -> Y1[a][u][r]
            dft8<false>(v);
            {
                const double2 w1 = Ws[u];  // w_1024^{u k} by recurrence (k <= 7)
                double2 wk = w1;
#pragma unroll
                for (int k = 1; k < 8; ++k) {
                    v[k] = c_mul(v[k], wk);
                    wk = c_mul(wk, w1);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) X[(k * 128 + u) * kRows + r] = v[k];
            __syncthreads();
            // PRM(s) and IDX(s+1) have been read by every thread: stage step s+1's
            if (more && tid == 0) stage_a(s + 1, s + 2);
            // stage 2: radix 8 over u2, twiddle w_128^{u1 b1} -> Y2[b1][a][u1][r]
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = X[(a8 * 128 + u1 + 16 * k) * kRows + r];
            __syncthreads();
            dft8<false>(v);
            {
                const double2 w1 = Ws[8 * u1];  // w_128^{u1 k} by recurrence
                double2 wk = w1;
#pragma unroll
                for (int k = 1; k < 8; ++k) {
                    v[k] = c_mul(v[k], wk);
                    wk = c_mul(wk, w1);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) X[((k * 8 + a8) * kPad + u1) * kRows + r] = v[k];
            __syncthreads();
            // stage 3: radix 16 over u1 = h + 2 i split over a lane pair (h = lane bit 2): each
            // half takes a radix 8 over i, the pair finishes with a radix 2 through shuffles;
            // then the four-step twiddle and the blocked store [rb][f][k1][8]
            {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = X[((b13 * 8 + a3) * kPad + h3 + 2 * i) * kRows + r];
                dft8<false>(v);
                if (h3) {  // E1[b] * w_16^b
#pragma unroll
                    for (int b = 1; b < 8; ++b) v[b] = c_mul(v[b], Ws[64 * b]);
                }
                mbar_wait(barZ, phZ);
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    // h = 0 keeps E0[b] + t_b (f-index b), h = 1 keeps E0[b] - t_b (b + 8)
                    const double2 o = make_double2(__shfl_xor_sync(0xffffffffu, v[b].x, 4),
                                                   __shfl_xor_sync(0xffffffffu, v[b].y, 4));
                    const double2 y = h3 ? c_sub(o, v[b]) : c_add(v[b], o);
                    const int f = a3 + 8 * b13 + 64 * (b + 8 * h3);
                    orow[(int64_t(f) * n1 + k1) * 8] = c_mul(y, Zs[f]);
                }
            }
            phZ ^= 1u;
            cp_wait_all();    // this thread's values(s+1) have landed
            __syncthreads();  // X and Z free
            if (more && tid == 0) stage_z(k1 - 1);
            if ((s & a.sync_mask) == a.sync_mask) cluster_sync();  // keep the row-block pair within a few steps
        }
    }
}

// The restart prologues of the fused pass as a separate, fully parallel pass: for every row
// and chain boundary k (k < 1024: chunk k's own upper end; k >= 1024: the midpoint of chunk
// k - 1024, where a split row block's second segment starts) the carry hchain_kernel would hold
// there -- carry = x_start, then the non-storing steps j = start-1 .. B-1 in its operand order.
// A warp is 32 consecutive rows of one boundary (512-byte gathers).  Replaces ~70 dependent
// gather steps per chunk at the start of every fused-pass unit.
__global__ void __launch_bounds__(256) p2fa_carry_kernel(const P2faArgs a, double2* __restrict__ carries) {
    const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int k = int(blockIdx.y);
    if (row >= a.rows) return;
    const int n1 = a.n1;
    const int c = k < kN ? k : k - kN;
    const int32_t start = k < kN ? __ldg(a.halo + c) : __ldg(a.halo_seg + 2 * c);
    const int64_t last = k < kN ? int64_t(c + 1) * n1 - 1 : int64_t(c) * n1 + n1 / 2 - 1;  // B - 1
    const double2* src = a.x1 + row;
    double2 carry = src[int64_t(__ldg(a.gather + start)) * a.ld];
    for (int64_t j = int64_t(start) - 1; j >= last; --j) {
        const double2 x = src[int64_t(__ldg(a.gather + j)) * a.ld];
        const double2 cs = __ldg(a.rec + 3 * j);
        carry = make_double2(__dadd_rn(__dmul_rn(cs.x, x.x), __dmul_rn(cs.y, carry.x)),
                             __dadd_rn(__dmul_rn(cs.x, x.y), __dmul_rn(cs.y, carry.y)));
    }
    carries[int64_t(k) * a.ldc + row] = carry;
}

// Step-major tables of one operator: rec_t[s][c] = {cs_j, d_{j+1}}, idx_t[s][c] = gather[j]
// for j = n1 c + n1 - 2 - s (zeros where j < 0).
__global__ void build_p2fa_tables_kernel(const double2* __restrict__ rec, const int32_t* __restrict__ gather, int n1,
                                         double2* rec_t, int32_t* idx_t) {
    const int c = int(blockIdx.x) * blockDim.x + threadIdx.x, s = int(blockIdx.y);
    if (c >= kN) return;
    const int64_t j = int64_t(n1) * c + (n1 - 2) - s;
    const size_t o = size_t(s) * kN + c;
    rec_t[2 * o] = j >= 0 ? rec[3 * j] : make_double2(0.0, 0.0);
    rec_t[2 * o + 1] = j >= 0 ? rec[3 * j + 2] : make_double2(0.0, 0.0);
    idx_t[o] = j >= 0 ? gather[j] : 0;
}

// z_t[k1][f] = w_n^{f k1} from the four-step tables (the product pass A forms per element)
__global__ void build_p2fa_twiddles_kernel(const double2* __restrict__ hi, const double2* __restrict__ lo, int shift,
                                           double2* z_t) {
    const int f = int(blockIdx.x) * blockDim.x + threadIdx.x, k1 = int(blockIdx.y);
    if (f >= kN) return;
    const int64_t e = int64_t(f) * k1;
    z_t[size_t(k1) * kN + f] = c_mul(hi[e >> shift], lo[e & ((int64_t(1) << shift) - 1)]);
}

}  // namespace

void build_p2fa_tables(const double2* rec, const int32_t* gather, int n1, double2* rec_t, int32_t* idx_t,
                       cudaStream_t stream) {
    build_p2fa_tables_kernel<<<dim3(kN / 256, n1), 256, 0, stream>>>(rec, gather, n1, rec_t, idx_t);
    MNB_LAUNCH_CHECK();
}

void build_p2fa_twiddles(const double2* hi, const double2* lo, int shift, int n1, double2* z_t, cudaStream_t stream) {
    build_p2fa_twiddles_kernel<<<dim3(kN / 256, n1), 256, 0, stream>>>(hi, lo, shift, z_t);
    MNB_LAUNCH_CHECK();
}

// chain chunks (= pass-B lengths) the fused pass and its pruned pass B cover: 128 (BASELINE c3,
// n = 2^17) ... 1024 (c4), and 3072 (c5)
bool p2fa_chunk_ok(int64_t n1) { return n1 == 128 || n1 == 256 || n1 == 512 || n1 == 1024 || n1 == 3072; }

// n = n1 x 1024 with pass A of length n2 = 1024 over the chunks and chain chunks of n1 indices
bool p2fa_supported(int64_t n, int64_t n1, int64_t n2, int64_t rows) {
    return n2 == kN && p2fa_chunk_ok(n1) && n == n1 * n2 && rows > 0 && rows % 8 == 0;
}

void launch_p2fa_carries(const P2faArgs& a, double2* carries, cudaStream_t stream) {
    const int64_t nrb = a.rows / 8;
    const int nb = std::min(a.full_rb, nrb) < nrb ? 2 * kN : kN;  // midpoints only when row blocks split
    p2fa_carry_kernel<<<dim3(ceil_div(a.rows, 256), unsigned(nb)), 256, 0, stream>>>(a, carries);
    MNB_LAUNCH_CHECK();
}

void launch_p2fa(const P2faArgs& a, int num_sms, cudaStream_t stream) {
    const size_t smem = P2faSmem::TOTAL;
    MNB_CUDA(cudaFuncSetAttribute(p2fa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int64_t nrb = a.rows / 8;
    const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(2 * nrb - std::min(a.full_rb, nrb), num_sms / 2));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(2 * pairs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MNB_CUDA(cudaLaunchKernelEx(&cfg, p2fa_kernel, a));
}

}  // namespace mnb
