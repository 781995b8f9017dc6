// Per-GPU context: stream, library handles, communicator, the (sharded)
// problem matrix, cached FFT plans and grow-only workspaces.
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <functional>
#include <map>
#include <memory>
#include <vector>

#include "common.cuh"
#include "host_srft.hpp"
#include "cholqr.cuh"
#include "kernels.cuh"
#include "pcg.cuh"

namespace mnb {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFree(p); }
    void* ensure(size_t need) {
        if (need > bytes) {
            if (p) MNB_CUDA(cudaFree(p));
            p = nullptr;
            bytes = 0;
            MNB_CUDA(cudaMalloc(&p, need));
            bytes = need;
        }
        return p;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() { if (p) cudaFreeHost(p); }
    void* ensure(size_t need) {
        if (need > bytes) {
            if (p) MNB_CUDA(cudaFreeHost(p));
            p = nullptr;
            bytes = 0;
            MNB_CUDA(cudaHostAlloc(&p, need, cudaHostAllocDefault));
            bytes = need;
        }
        return p;
    }
};

// Device-side FFT plan for one length n (four-step or single pass).
struct FftLenPlan {
    int N = 1, E = 1, nradix = 0, radix[10] = {0};
    bool direct = false;
    DevBuf tw;  // w_N^q
};
struct FftPlan {
    int64_t n = 0, n1 = 1, n2 = 1;  // n = n1 * n2 ; pass A length n2 (batches n1), pass B length n1
    bool single = true;
    FftLenPlan A, B;                 // single: only A (N = n)
    DevBuf tw4_hi, tw4_lo;
    int tw4_shift = 0;
    DevBuf p2fa_z;  // fused H + pass A: w_n^{f k1} per k1 row (built on first use)
};

// Device copy of one operator's parameter blob (layout of SrftHost).
struct SrftDev {
    const SrftHost* host = nullptr;
    DevBuf blob;
    DevBuf dups;
    int64_t ndups = 0;
    DevBuf chain_rec[2];  // per-step chain records of the sketch H stages: [0] P1 (tilde half), [1] P2
    DevBuf vec_halo;      // restart points of 64-index chunks for single-vector chains: fwd, fwd~, adj, adj~
    int64_t vec_chunk = 0, vec_nchunks = 0;
    DevBuf p2fa_rec, p2fa_idx, p2fa_halo;  // + restart points of 512-index sub-chunks (fwd, adj)  // fused H + pass A: step-major chain records / gather indices (n = 2^20)
    DevBuf fb_csr;        // kept frequencies per f2 for the pruned FFT pass B: [n2+1 offsets][(f1, slot) pairs]
    int64_t fb_n2 = 0;
    // page-locked staging of the small host-built tables (dups, fb_csr): async uploads, no
    // pageable copies (which serialise the host behind the stream)
    PinnedBuf stage;
    cudaEvent_t stage_free = nullptr;  // the last upload out of `stage` has completed
    SrftDev() = default;
    SrftDev(const SrftDev&) = delete;
    SrftDev& operator=(const SrftDev&) = delete;
    ~SrftDev() { if (stage_free) cudaEventDestroy(stage_free); }
    template <class T> const T* at(size_t off) const { return reinterpret_cast<const T*>(blob.as<unsigned char>() + off); }
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    cublasHandle_t cublas = nullptr;
    cusolverDnHandle_t cusolver = nullptr;
    cusolverDnParams_t cusolver_params = nullptr;
    ncclComm_t comm = nullptr;  // set by mnb_context_create_distributed (any world size, 1 included)
    int rank = 0, world = 1;
    bool distributed() const { return comm != nullptr; }

    // problem matrix (this rank's column shard)
    int dtype = MNB_C128;
    int64_t m = 0, n_global = 0, col_begin = 0, n_local = 0;
    const void* A = nullptr;
    DevBuf A_own;
    // deferred host copy (MNB_HOST_ASYNC): A_own is allocated, the bytes are still on the host
    const void* A_host = nullptr;
    int64_t host_lda = 0;
    bool pending_host = false;
    cudaStream_t copy_stream = nullptr;

    std::map<int64_t, std::unique_ptr<FftPlan>> fft_plans;
    int64_t launches = 0;  // own kernels launched (for reporting)

    // workspaces
    DevBuf ws_x1, ws_x2, ws_slab, ws_pack, ws_carry;
    // distributed: this rank's row block of A after the all-to-all (redistribute_rows), valid
    // until the matrix changes or the next solve starts
    bool slab_ready = false;
    int64_t slab_rows = 0, slab_row0 = 0;
    DevBuf sk_S, sk_E, tau_S, tau_E, qr_work, qr_info, R_S, R_E, R2, gram, qwork, gram_E, gram_Sk;
    cudaStream_t gram_stream = nullptr;  // E's Gram built slab by slab beside the sketch
    bool init_from_sketch = false;  // this solve's CG INIT took A c = S^H z (no pass over A)
    // multi-slab sketches: called after each row slab's kernels are queued (rows [s0, s0 + rs) of
    // the output are final once they run); the solve uses it to build E's Gram block by block
    std::function<void(int64_t s0, int64_t rs)> on_slab;
    // staged operator upload: called once by sketch_block right after the first H stage of the
    // first slab is queued (the operator's other half is then uploaded behind it)
    std::function<void()> after_first_stage;
    const double2* pre_gram = nullptr;  // when set, the next CholeskyQR pass 1 takes this S^H S (upper)
    bool qr_shifted = false;  // this solve's first sketch needed shifted CholeskyQR3 (reset per solve)
    bool p2fa = true;    // fused P2 + FFT pass A (k_p2fa.cu) where the shape allows; MNB_P2FA=0 disables
    bool two_norm_check = true;  // one-pass preconditioner accepted on a 2-norm cond estimate; MNB_PRECOND_2NORM=0 disables
    bool csne = true;    // Step 2 from R1 = chol(S^H S) + corrected seminormal equations; MNB_CSNE=0 disables
    bool cholqr = true;  // CholeskyQR2 for the sketch QRs (Householder fallback); MNB_QR=householder disables
    // the sketch QRs on the hand-written kernels (k_cholqr.cu): Cholesky, triangular inverse and the
    // device-resident Step-2 / preconditioner-check loops, one host read per sketch.
    // MNB_FASTQR=0: the host-steered chain of cholqr_r; MNB_QR_LIB=1: cuSOLVER potrf + ZTRSM inverse
    bool fastqr = true;
    bool qr_lib = false;
    DevBuf qr_status, qr_part, tri_work, tri_x1;
    const double2* gram0 = nullptr;  // this sketch's Gram S^H S kept beside the one-pass Cholesky (shifted two-pass chain)
    PinnedBuf pin_qr, pin_vec;  // status mirror; page-locked staging of b and the power-step start vector
    DevBuf Rinv, Rinv_rows;
    DevBuf vec_m[12], vec_n[4], vec_full[3], red, part_s, part_scal, part_gg, part_gg_init, state, resid, scratch;
    DevBuf rhs, flag, out_c, qprobe;
    int* nonfinite = nullptr;  // set while sketching the problem matrix (finiteness check)
    PinnedBuf pin_params[2], pin_small;
    struct SlabCache {
        int64_t n = -1, rows = -1, l = -1, m = -1, Ms = 0;
    } slab_cache;  // sketch slab height per shape (srft_gpu.cu sketch_block)
    SrftDev op_dev[3];  // device copies of the operators: [0] T, [1] T', [2] standalone SRFT calls (grow-only)
    std::vector<cudaEvent_t> events;
    // deferred kernel timers (EventTimer): event pool + pending (start, stop, accumulator)
    struct PendingTimer {
        cudaEvent_t a, b;
        double* acc;
    };
    std::vector<cudaEvent_t> timer_pool;
    size_t timer_next = 0;
    std::vector<PendingTimer> timers;
    cudaStream_t aux_stream = nullptr;  // second compute stream (QRs / Steps 2-3 beside the sketches and passes)
    // QR(E) runs on a host helper thread with its own stream, library handles and workspaces
    // (beside QR(S) / Steps 2-3, which hold host round trips of their own): created on first use
    std::unique_ptr<Context> qr_helper;
    Context& helper();
    std::vector<unsigned char> host_work;  // cuSOLVER host workspace (kept alive across async calls)

    ~Context();
    cudaEvent_t event(size_t i);
    cudaEvent_t timer_event();
    void resolve_timers();  // synchronizes on the pending timers and accumulates them
    FftPlan& fft_plan(int64_t n);
    size_t esz() const { return dtype == MNB_F64 ? 8 : 16; }
    void make_resident();  // completes a deferred host copy of A (synchronous)
};

// ---- SRFT on the GPU (srft_gpu.cu) ----
void upload_srft(Context& ctx, const SrftHost& op, SrftDev& dev);
void upload_srft_first(Context& ctx, const SrftHost& op, SrftDev& dev);
void upload_srft_rest(Context& ctx, const SrftHost& op, SrftDev& dev, cudaStream_t side, cudaEvent_t landed);
// T * conj(rows [row0,row0+rows) of a column-major block) -> out[slot + (out_row0 + r) * ldo]
void sketch_block(Context& ctx, const SrftDev& op, const void* Ablk, int is_real, int64_t lda, int64_t row0,
                  int64_t rows, double2* out, int64_t ldo, int64_t out_row0, double* kernel_ms);
// The sketch all-to-all's table (see mnb_redistribute_plan) and the exchange itself.
void redistribute_plan(int64_t m, int64_t n_global, int world, int rank, int64_t* plan);
void redistribute_rows(Context& ctx, double* seconds);
// Full sketch of the context matrix (distributed: local rows of the redistributed slab +
// allgather; the all-to-all runs first if this solve has not done it): out l x m col-major (device).
void sketch_matrix(Context& ctx, const SrftDev& op, double2* out, double* kernel_ms, double* redistribute_s);
// T^* v for one device vector v (l) -> y (n, device).
void srft_adjoint_vec(Context& ctx, const SrftDev& op, const double2* v, double2* y);
// T x / H x for one device vector.
void srft_apply_vec(Context& ctx, const SrftDev& op, const double2* x, double2* y, bool h_only);
void dft_vec(Context& ctx, int64_t n, double2* x, bool inverse);

// ---- solver (solver.cu) ----
struct LsqResult {
    int64_t iterations = 0;
    bool converged = false;
    double achieved_excess = 0.0;
    double rr0 = 0.0;
    double xx = 0.0;  // ||x||^2 when run_cg accumulated x
    std::vector<double> residual_norms;
    double pass_ms = 0.0;
    int64_t pass_launches = 0;
    double pcg_seconds = 0.0;
};
void sync(Context& ctx);
void trace(const char* what);  // MNB_TRACE=1: host phase timestamps on stderr
// a secondary context on the same device (abi.cu): own stream, cuBLAS / cuSOLVER handles
std::unique_ptr<Context> make_helper_context(const Context& parent);
void solve_randomized(Context& ctx, const double2* b_host, const mnb_solver_config& cfg, double2* x_dev,
                      double2* c_dev, mnb_solve_report& rep);
void solve_classical(Context& ctx, const double2* b_host, double2* x_dev, mnb_classical_report& rep);
void apply_adjoint_matrix(Context& ctx, const void* y, bool y_on_device, double2* x_dev, double2* ax_host);
void solve_least_squares(Context& ctx, const double2* c_dev, const mnb_lsq_config& cfg, double2* y_host,
                         double* residual_norms, mnb_lsq_solution& sol);
double bench_pcg_pass(Context& ctx, int reps);
// Step 2 on a host sketch (mnb_csne_solve): Gram, Cholesky, inverse, corrected seminormal equations
void csne_solve_host(Context& ctx, const double2* S, int64_t l, int64_t m, const double2* b, double2* z,
                     double* status);

}  // namespace mnb
