// The randomized minimal-norm solve on the GPU (src/solver.cpp:50-128) and
// its least-squares subsolver (src/lsq.cpp:43-113).
//
//   Step 1  S = T·A^H                     sketch_matrix  (SRFT kernels)
//   Step 2  S = QR, z = Q [R^{-H} b; 0]    cuSOLVER geqrf / cuBLAS trsv / unmqr
//   Step 3  c = T^* z                      srft_adjoint_vec
//   Step 4  E = T'·A^H, E = Q'R', CG on the normal equations of A^H R'^{-1}
//           (fused pass kernel, explicit R'^{-1} from trtri, device-side loop)
//   Step 5  x = A^H y, ||A x - b||         one more fused pass
//
// Multi-GPU (column-sharded A): one NCCL allreduce of [s, qq, <r,t>, ||r||^2]
// (2m+4 doubles) per CG iteration; the sketch redistributes A with one
// all-to-all (srft_gpu.cu).  The small m-space work is replicated per rank.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <future>
#include <thread>

#include "context.cuh"

namespace mnb {

namespace {

constexpr double kEps = 2.220446049250313080847e-16;

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}


void cusolver_check(cusolverStatus_t s, const char* what) {
    if (s != CUSOLVER_STATUS_SUCCESS) throw Error(MNB_ERR_CUDA, std::string(what) + " failed (cusolver status " + std::to_string(int(s)) + ")");
}
void cublas_check(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) throw Error(MNB_ERR_CUDA, std::string(what) + " failed (cublas status " + std::to_string(int(s)) + ")");
}
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(MNB_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

template <class T>
T* dev(DevBuf& b, size_t count) {
    return static_cast<T*>(b.ensure(count * sizeof(T) + 16));
}

// Householder QR of the tall l x m sketch in place (Eigen::HouseholderQR at
// src/solver.cpp:86 and src/lsq.cpp:58; LAPACK/cuSOLVER use the same
// reflector convention R_jj = -sign(Re x0)||x||).
void qr_in_place(Context& ctx, double2* S, int64_t l, int64_t m, double2* tau) {
    size_t dws = 0, hws = 0;
    cusolver_check(cusolverDnXgeqrf_bufferSize(ctx.cusolver, ctx.cusolver_params, l, m, CUDA_C_64F, S, l, CUDA_C_64F,
                                               tau, CUDA_C_64F, &dws, &hws),
                   "geqrf_bufferSize");
    void* work = ctx.qr_work.ensure(std::max<size_t>(dws, 16));
    if (ctx.host_work.size() < hws + 16) ctx.host_work.resize(hws + 16);
    int* info = dev<int>(ctx.qr_info, 1);
    cusolver_check(cusolverDnXgeqrf(ctx.cusolver, ctx.cusolver_params, l, m, CUDA_C_64F, S, l, CUDA_C_64F, tau,
                                    CUDA_C_64F, work, dws, ctx.host_work.data(), hws, info),
                   "geqrf");
}

// src/lsq.cpp:18-27 / src/solver.cpp:25-33: entries |R_jj| < rows*eps*max|R_jj| (or exactly 0).
int64_t deficient_count(Context& ctx, const double2* QR, int64_t ld, int64_t m, int64_t rows) {
    std::vector<double> diag(size_t(2 * m));
    MNB_CUDA(cudaMemcpy2DAsync(diag.data(), 16, QR, size_t(ld + 1) * 16, 16, size_t(m), cudaMemcpyDeviceToHost,
                               ctx.stream));
    MNB_CUDA(cudaStreamSynchronize(ctx.stream));
    double dmax = 0.0;
    for (int64_t j = 0; j < m; ++j) dmax = std::max(dmax, std::hypot(diag[size_t(2 * j)], diag[size_t(2 * j + 1)]));
    const double thr = double(rows) * kEps * dmax;
    int64_t bad = 0;
    for (int64_t j = 0; j < m; ++j) {
        const double re = diag[size_t(2 * j)], im = diag[size_t(2 * j + 1)];
        if (std::hypot(re, im) < thr || (re == 0.0 && im == 0.0)) ++bad;
    }
    return bad;
}

void allreduce_sum(Context& ctx, double* buf, size_t count) {
    if (ctx.distributed())
        nccl_check(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx.comm, ctx.stream), "ncclAllReduce");
}

struct PassBuffers {
    PcgPlan plan;
    double2 *part_s;
    double *part_scal, *red;
};

PassBuffers pass_buffers(Context& ctx) {
    PassBuffers b;
    b.plan = plan_pcg_pass(ctx.m, std::max<int64_t>(ctx.n_local, 1), ctx.dtype == MNB_F64, ctx.num_sms);
    // (sized for the persistent small-CG kernel's partials too, so that path never regrows -- and
    // frees -- these buffers under a queued pass)
    const size_t parts = std::max<size_t>(size_t(b.plan.grid),
                                          size_t(pcg_small_grid(ctx.m, std::max<int64_t>(ctx.n_local, 1), ctx.num_sms)));
    b.part_s = dev<double2>(ctx.part_s, parts * size_t(ctx.m));
    b.part_scal = dev<double>(ctx.part_scal, parts * 4);
    b.red = dev<double>(ctx.red, size_t(2 * ctx.m + 4));
    return b;
}

// One fused pass + deterministic reduction (+ allreduce across ranks).
void fused_pass(Context& ctx, const PassBuffers& pb, int mode, const double2* w, const double2* tin, double2* tout,
                double2* r, const CgState* state, double2* x = nullptr) {
    if (ctx.n_local > 0) {
        PcgPassArgs a;
        a.A = ctx.A;
        a.is_real = ctx.dtype == MNB_F64;
        a.m = ctx.m;
        a.n = ctx.n_local;
        a.w = w;
        a.tin = tin;
        a.tout = tout;
        a.r = r;
        a.x = x;
        a.state = state;
        a.part_s = pb.part_s;
        a.part_scal = pb.part_scal;
        a.mode = mode;
        launch_pcg_pass(a, pb.plan, ctx.stream);
        launch_pcg_reduce(pb.part_s, pb.part_scal, pb.plan.grid, ctx.m, pb.red, state, ctx.stream);
        ctx.launches += 2;
    } else {
        MNB_CUDA(cudaMemsetAsync(pb.red, 0, size_t(2 * ctx.m + 4) * 8, ctx.stream));
    }
    allreduce_sum(ctx, pb.red, size_t(2 * ctx.m + 4));
}

}  // namespace

// Rinv = R^{-1} for the upper-triangular m x m R (leading dimension ldR), the CG's explicit
// preconditioner; the strictly lower triangle of Rinv comes out zero.  MNB_QR_LIB=1: one
// tensor-core ZTRSM against the identity (or MNB_TRTRI=1: cuSOLVER Xtrtri, ~2x slower at m = 2048).
void upper_inverse(Context& ctx, const double2* R, int64_t ldR, int64_t m, double2* Rinv, CholStatus* st = nullptr) {
    if (!ctx.qr_lib) {  // the hand-written blocked inverse (k_cholqr.cu); st->xnorm2 = ||Rinv||_F^2
        double2* W = dev<double2>(ctx.tri_work, size_t(m) * size_t(m));
        launch_trtri_upper(R, ldR, m, Rinv, W, st, ctx.num_sms, ctx.stream, /*gate_on_chol=*/st != nullptr);
        ctx.launches += 1;
        return;
    }
    static const bool use_trtri = [] { const char* e = std::getenv("MNB_TRTRI"); return e && std::string(e) == "1"; }();
    if (use_trtri) {
        MNB_CUDA(cudaMemcpy2DAsync(Rinv, size_t(m) * 16, R, size_t(ldR) * 16, size_t(m) * 16, size_t(m),
                                   cudaMemcpyDeviceToDevice, ctx.stream));
        size_t dws = 0, hws = 0;
        cusolver_check(cusolverDnXtrtri_bufferSize(ctx.cusolver, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, m,
                                                   CUDA_C_64F, Rinv, m, &dws, &hws),
                       "trtri_bufferSize");
        void* work = ctx.qr_work.ensure(std::max<size_t>(dws, 16));
        if (ctx.host_work.size() < hws + 16) ctx.host_work.resize(hws + 16);
        cusolver_check(cusolverDnXtrtri(ctx.cusolver, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, m, CUDA_C_64F, Rinv,
                                        m, work, dws, ctx.host_work.data(), hws, dev<int>(ctx.qr_info, 1)),
                       "trtri");
        return;
    }
    MNB_CUDA(cudaMemsetAsync(Rinv, 0, size_t(m) * size_t(m) * 16, ctx.stream));
    launch_add_diagonal(Rinv, m, 1.0, ctx.stream);
    ctx.launches += 1;
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
    cublas_check(cublasZtrsm(ctx.cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                             int(m), int(m), &one, reinterpret_cast<const cuDoubleComplex*>(R), int(ldR),
                             reinterpret_cast<cuDoubleComplex*>(Rinv), int(m)),
                 "ztrsm");
}

// MNB_TRACE=1: host timestamps of the solve's phases on stderr (diagnostics)
void trace(const char* what) {
    static const bool on = std::getenv("MNB_TRACE") != nullptr;
    if (!on) return;
    static thread_local double last = 0.0;
    const double t = now_s();
    std::fprintf(stderr, "[mnb] %-28s +%8.3f ms\n", what, last > 0.0 ? (t - last) * 1e3 : 0.0);
    last = t;
}

void sync(Context& ctx) { MNB_CUDA(cudaStreamSynchronize(ctx.stream)); }

// MNB_TRACE=1: device-side stage times of one stream (events between the stages; dump() waits
// for the last one and prints the gaps).  Off: no events, no cost.
struct DevTrace {
    Context& ctx;
    const char* what;
    bool on;
    std::vector<std::pair<const char*, cudaEvent_t>> marks;
    DevTrace(Context& c, const char* w) : ctx(c), what(w), on(std::getenv("MNB_TRACE") != nullptr) { mark("start"); }
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        MNB_CUDA(cudaEventCreate(&e));
        MNB_CUDA(cudaEventRecord(e, ctx.stream));
        marks.emplace_back(name, e);
    }
    void dump() {
        if (!on || marks.empty()) return;
        MNB_CUDA(cudaEventSynchronize(marks.back().second));
        std::string line = std::string("[mnb] device ") + what + ":";
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            MNB_CUDA(cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second));
            char buf[96];
            std::snprintf(buf, sizeof buf, " %s %.3f", marks[i].first, ms);
            line += buf;
        }
        std::fprintf(stderr, "%s ms\n", line.c_str());
        for (auto& m : marks) cudaEventDestroy(m.second);
        marks.clear();
    }
    ~DevTrace() {
        for (auto& m : marks) cudaEventDestroy(m.second);
    }
};

Context::~Context() {
    for (auto e : events) if (e) cudaEventDestroy(e);
    for (auto e : timer_pool) if (e) cudaEventDestroy(e);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    if (cusolver_params) cusolverDnDestroyParams(cusolver_params);
    if (cusolver) cusolverDnDestroy(cusolver);
    if (cublas) cublasDestroy(cublas);
    if (comm) ncclCommDestroy(comm);
    if (own_stream && stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (gram_stream) cudaStreamDestroy(gram_stream);
}

void Context::make_resident() {
    if (!pending_host) return;
    const size_t e = esz();
    MNB_CUDA(cudaMemcpy2DAsync(A_own.p, size_t(m) * e, A_host, size_t(host_lda) * e, size_t(m) * e, size_t(n_local),
                               cudaMemcpyHostToDevice, stream));
    MNB_CUDA(cudaStreamSynchronize(stream));
    pending_host = false;
    A_host = nullptr;
}

Context& Context::helper() {
    if (!qr_helper) qr_helper = make_helper_context(*this);
    qr_helper->m = m;
    return *qr_helper;
}

cudaEvent_t Context::timer_event() {
    if (timer_next == timer_pool.size()) {
        cudaEvent_t e;
        MNB_CUDA(cudaEventCreate(&e));
        timer_pool.push_back(e);
    }
    return timer_pool[timer_next++];
}

void Context::resolve_timers() {
    for (const auto& t : timers) {
        MNB_CUDA(cudaEventSynchronize(t.b));
        float ms = 0.f;
        MNB_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
        *t.acc += ms;
    }
    timers.clear();
    timer_next = 0;
}

cudaEvent_t Context::event(size_t i) {
    while (events.size() <= i) {
        cudaEvent_t e;
        MNB_CUDA(cudaEventCreate(&e));
        events.push_back(e);
    }
    return events[i];
}

// ------------------------------------------------------------- CG loop ----
// solve_least_squares (src/lsq.cpp:43-113) from the sketch R' onward.
// c: this rank's n_local entries (device).  y: m entries (device).
// x, ax (optional): also accumulate x = A^H y = sum_k alpha_k t_k (this rank's columns) and
// A x = sum_k alpha_k s_k inside the CG passes, so Step 5 (src/solver.cpp:118-125) needs no extra pass.
// The INIT pass of the CG (lsq.cpp:77-86: r = c, s = A c, ||c||^2) on ctx.stream.  It needs only c,
// so the solve launches it ahead of the preconditioner's QR (run_cg with init_done).
void launch_cg_init_pass(Context& ctx, const double2* c, double2* x) {
    const int64_t n = ctx.n_local;
    double2* r = dev<double2>(ctx.vec_n[0], size_t(std::max<int64_t>(n, 1)));
    double2* t = dev<double2>(ctx.vec_n[1], size_t(std::max<int64_t>(n, 1)));
    PassBuffers pb = pass_buffers(ctx);
    MNB_CUDA(cudaEventRecord(ctx.event(20), ctx.stream));
    fused_pass(ctx, pb, PCG_INIT, nullptr, c, t, r, nullptr, x);
    MNB_CUDA(cudaEventRecord(ctx.event(21), ctx.stream));
}

// The same INIT without touching A, for the solve (one GPU): c = T^* z is Step 3's output, so
// A c = A T^* z = (T A^*)^* z = S^H z -- one l x m GEMV over the sketch (256 MiB at c4) in place
// of a 32 GiB pass.  In exact arithmetic S^H z = b (c solves A c = b); the computed S^H z carries
// the same u ||S|| ||z|| rounding as a direct A c, so the CG's g_0 = R'^{-H} A c is as accurate.
void launch_cg_init_from_sketch(Context& ctx, const double2* S, int64_t l, const double2* z, const double2* c,
                                double2* x) {
    const int64_t n = ctx.n_local, m = ctx.m;
    double2* r = dev<double2>(ctx.vec_n[0], size_t(std::max<int64_t>(n, 1)));
    double2* t = dev<double2>(ctx.vec_n[1], size_t(std::max<int64_t>(n, 1)));
    PassBuffers pb = pass_buffers(ctx);
    const int parts = 4 * ctx.num_sms;
    double* part = dev<double>(ctx.part_gg_init, size_t(parts));
    MNB_CUDA(cudaEventRecord(ctx.event(20), ctx.stream));
    launch_sketch_adjoint_gemv(S, l, m, z, reinterpret_cast<double2*>(pb.red), ctx.stream);
    launch_cg_init_vectors(c, n, r, t, x, part, parts, pb.red + 2 * m, ctx.stream);
    ctx.launches += 3;
    allreduce_sum(ctx, pb.red + 2 * m, 4);  // ||c||^2 over the ranks' columns (S^H z is already global)
    MNB_CUDA(cudaEventRecord(ctx.event(21), ctx.stream));
    ctx.init_from_sketch = true;
}

LsqResult run_cg(Context& ctx, const double2* c, const double2* Rtop, int64_t ldR, double tau, int64_t max_it,
                 double dup, double2* y, bool want_norms, double2* x, double2* ax, bool init_done,
                 bool rinv_ready, const double2* rinv_src = nullptr) {
    const int64_t m = ctx.m, n = ctx.n_local;
    LsqResult res;
    const double t0 = now_s();
    // explicit R'^{-1} (consistent forward/adjoint preconditioner)
    double2* Rinv = dev<double2>(ctx.Rinv, size_t(m) * size_t(m));
    double2* Rinv_rows = dev<double2>(ctx.Rinv_rows, size_t(m) * size_t(m));
    if (!rinv_ready) upper_inverse(ctx, Rtop, ldR, m, Rinv);  // (else the one-pass Cholesky path left it)
    else if (rinv_src && rinv_src != Rinv)  // ... in the helper context's buffer
        MNB_CUDA(cudaMemcpyAsync(Rinv, rinv_src, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
    launch_transpose(Rinv, m, m, m, Rinv_rows, m, ctx.stream);
    ctx.launches += 1;

    double2* w = dev<double2>(ctx.vec_m[0], size_t(m));
    double2* u = dev<double2>(ctx.vec_m[1], size_t(m));
    double2* g = dev<double2>(ctx.vec_m[2], size_t(m));
    double2* dir = dev<double2>(ctx.vec_m[3], size_t(m));
    double2* dir_old = dev<double2>(ctx.vec_m[4], size_t(m));
    double2* r = dev<double2>(ctx.vec_n[0], size_t(std::max<int64_t>(n, 1)));
    double2* t = dev<double2>(ctx.vec_n[1], size_t(std::max<int64_t>(n, 1)));
    CgState* st = dev<CgState>(ctx.state, 1);
    double* norms = dev<double>(ctx.resid, size_t(max_it + 2));
    const int ub = pcg_upd_blocks(m);
    double* part_gg = dev<double>(ctx.part_gg, size_t(ub));
    PassBuffers pb = pass_buffers(ctx);

    launch_init_state(st, tau, dup, (long long)max_it, ctx.stream);
    // initial state (lsq.cpp:77-86): r = c, g = M^H c, dir = g
    cudaEvent_t ea = ctx.event(20), eb = ctx.event(21);
    if (!init_done) launch_cg_init_pass(ctx, c, x);
    launch_pcg_upd1(pb.red, Rinv, m, u, g, dir, dir_old, part_gg, st, norms, 1, ctx.stream, ax);
    launch_pcg_upd2(part_gg, ub, Rinv_rows, m, g, dir_old, dir, w, st, 1, ctx.stream);
    ctx.launches += 3;

    int* done_h = static_cast<int*>(ctx.pin_small.ensure(sizeof(CgState) + 64));
    CgState* st_h = reinterpret_cast<CgState*>(done_h);
    auto read_state = [&]() {
        MNB_CUDA(cudaMemcpyAsync(st_h, st, sizeof(CgState), cudaMemcpyDeviceToHost, ctx.stream));
        MNB_CUDA(cudaStreamSynchronize(ctx.stream));
    };
    // CG iterations (lsq.cpp:88-107).  L2-resident A on one GPU: the whole loop is one persistent
    // cooperative kernel (k_pcg_small.cu); otherwise K iterations of (pass, reduce, upd1, upd2)
    // between host polls of the device-side done flag (kernels of finished loops exit at once).
    const int64_t K = 4;
    int64_t issued = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pass_ev;
    const bool small = !ctx.distributed() && n > 0 && pcg_small_eligible(m, n, ctx.dtype == MNB_F64) &&
                       !std::getenv("MNB_SMALL_CG_OFF");
    if (small) {
        SmallCgArgs a;
        a.A = ctx.A;
        a.is_real = ctx.dtype == MNB_F64;
        a.m = m;
        a.n = n;
        a.Rinv = Rinv;
        a.Rinv_rows = Rinv_rows;
        a.u = u;
        a.g = g;
        a.dir = dir;
        a.dir_old = dir_old;
        a.w = w;
        a.ax = ax;
        a.r = r;
        a.t = t;
        a.x = x;
        const int grid = pcg_small_grid(m, n, ctx.num_sms);
        a.part_s = dev<double2>(ctx.part_s, size_t(grid) * size_t(m));
        a.part_scal = dev<double>(ctx.part_scal, size_t(grid) * 4);
        a.s = reinterpret_cast<double2*>(pb.red);
        a.part_gg = dev<double>(ctx.part_gg, size_t(std::max(grid, ub)));
        a.st = st;
        a.residual_norms = norms;
        cudaEvent_t e0 = ctx.event(32), e1 = ctx.event(33);
        MNB_CUDA(cudaEventRecord(e0, ctx.stream));
        launch_pcg_small(a, grid, ctx.stream);
        MNB_CUDA(cudaEventRecord(e1, ctx.stream));
        ctx.launches += 1;
        pass_ev.emplace_back(e0, e1);
    }
    // one GPU, A beyond L2: each iteration is the fused pass + one cooperative update launch
    // (k_pcg_small.cu pcg_update_kernel) in place of reduce / upd1 / upd2; multi-GPU keeps the
    // three kernels around the per-iteration allreduce
    // (distributed: pass + reduce + allreduce, then the update kernel on the allreduced vector)
    const bool merged = !small && n > 0 && !std::getenv("MNB_CG_UPD3");
    const int ugrid = pcg_update_grid(m, ctx.num_sms);
    SmallCgArgs ua;
    if (merged) {
        ua.m = m;
        ua.Rinv = Rinv;
        ua.Rinv_rows = Rinv_rows;
        ua.u = u;
        ua.g = g;
        ua.dir = dir;
        ua.dir_old = dir_old;
        ua.w = w;
        ua.ax = ax;
        ua.part_s = pb.part_s;
        ua.part_scal = pb.part_scal;
        ua.s = reinterpret_cast<double2*>(pb.red);
        ua.part_gg = dev<double>(ctx.part_gg, size_t(std::max(ugrid, ub)));
        ua.st = st;
        ua.residual_norms = norms;
    }
    auto launch_pass_only = [&](int mode) {
        PcgPassArgs a;
        a.A = ctx.A;
        a.is_real = ctx.dtype == MNB_F64;
        a.m = m;
        a.n = n;
        a.w = w;
        a.tin = t;
        a.tout = t;
        a.r = r;
        a.x = x;
        a.state = st;
        a.part_s = pb.part_s;
        a.part_scal = pb.part_scal;
        a.mode = mode;
        launch_pcg_pass(a, pb.plan, ctx.stream);
    };
    for (; !small;) {
        read_state();
        if (st_h->done || issued >= max_it + 1) break;
        for (int64_t k = 0; k < K; ++k) {
            cudaEvent_t e0 = ctx.event(32 + 2 * size_t(issued)), e1 = ctx.event(33 + 2 * size_t(issued));
            if (merged && !ctx.distributed()) {  // the pass, then reduce + gradient + direction in one launch
                MNB_CUDA(cudaEventRecord(e0, ctx.stream));
                launch_pass_only(PCG_CG);
                MNB_CUDA(cudaEventRecord(e1, ctx.stream));
                launch_pcg_update(ua, pb.plan.grid, ugrid, ctx.stream);
                ctx.launches += 2;
            } else if (merged) {  // pass + reduce + allreduce, then gradient + direction in one launch
                MNB_CUDA(cudaEventRecord(e0, ctx.stream));
                fused_pass(ctx, pb, PCG_CG, w, t, t, r, st, x);
                MNB_CUDA(cudaEventRecord(e1, ctx.stream));
                launch_pcg_update(ua, 0, ugrid, ctx.stream);
                ctx.launches += 1;
            } else {
                MNB_CUDA(cudaEventRecord(e0, ctx.stream));
                fused_pass(ctx, pb, PCG_CG, w, t, t, r, st, x);
                MNB_CUDA(cudaEventRecord(e1, ctx.stream));
                launch_pcg_upd1(pb.red, Rinv, m, u, g, dir, dir_old, part_gg, st, norms, 0, ctx.stream, ax);
                launch_pcg_upd2(part_gg, ub, Rinv_rows, m, g, dir_old, dir, w, st, 0, ctx.stream);
                ctx.launches += 2;
            }
            pass_ev.emplace_back(e0, e1);
            ++issued;
        }
    }
    // exact final residual and y = R'^{-1} u (lsq.cpp:109-111)
    double* scratch = dev<double>(ctx.scratch, 1024);
    if (n > 0) {
        launch_pcg_finalize(r, t, x, n, st, scratch, ctx.stream);
        ctx.launches += 2;
    } else {
        MNB_CUDA(cudaMemsetAsync(&st->rr_final, 0, 16, ctx.stream));
    }
    allreduce_sum(ctx, &st->rr_final, 2);  // rr_final, xx_final
    launch_trmv_rows(Rinv_rows, m, u, y, ctx.stream);
    ctx.launches += 1;
    read_state();
    res.iterations = st_h->iterations;
    res.converged = st_h->converged != 0;
    res.rr0 = st_h->rr0;
    res.xx = st_h->xx_final;
    const double rr = st_h->rr_final, excess = st_h->excess;
    const double min_est = std::max(rr - excess, 0.0);
    res.achieved_excess = min_est > 0.0 ? excess / min_est : 0.0;
    // device time of the passes that did work: the INIT pass + one per iteration
    float ms = 0.f;
    MNB_CUDA(cudaEventElapsedTime(&ms, ea, eb));
    res.pass_ms = ctx.init_from_sketch ? 0.f : ms;  // (the INIT pass, when there was one)
    res.pass_launches = ctx.init_from_sketch ? 0 : 1;
    ctx.init_from_sketch = false;
    if (small) {  // one launch for the whole loop: report it per iteration
        MNB_CUDA(cudaEventElapsedTime(&ms, pass_ev[0].first, pass_ev[0].second));
        res.pass_ms += ms;
        res.pass_launches += std::max<int64_t>(1, res.iterations);
    }
    const int64_t worked =
        small ? 0 : std::min<int64_t>(int64_t(pass_ev.size()), res.iterations + (st_h->stop_qq0 ? 1 : 0));
    for (int64_t i = 0; i < worked; ++i) {
        MNB_CUDA(cudaEventElapsedTime(&ms, pass_ev[size_t(i)].first, pass_ev[size_t(i)].second));
        res.pass_ms += ms;
        res.pass_launches += 1;
    }
    if (want_norms) {
        res.residual_norms.resize(size_t(res.iterations + 1));
        MNB_CUDA(cudaMemcpy(res.residual_norms.data(), norms, size_t(res.iterations + 1) * 8, cudaMemcpyDeviceToHost));
        res.residual_norms[size_t(res.iterations)] = std::sqrt(rr);
    }
    res.pcg_seconds = now_s() - t0;
    return res;
}

// ------------------------------------------------------------- helpers ----
struct SketchQr {
    double2* S;         // the sketch (Householder path: overwritten by geqrf's reflectors and R)
    double2* tau;       // Householder path only
    const double2* R;   // m x m upper triangle, leading dimension ldR
    int64_t ldR;
    bool householder;
    int path = 0;       // 0 CholeskyQR2, 1 shifted CholeskyQR3, 2 Householder, 3 one Cholesky pass (preconditioner)
    bool rinv_ready = false;  // path 3: R^{-1} already in ctx.Rinv
    int64_t deficient = -1;   // the rank rule's count when the Cholesky kernel already took it (else -1)
};

// CholeskyQR2 of the l x m sketch, R only (S is left intact) -- or, for sketches too ill-
// conditioned for it, shifted CholeskyQR3 (a diagonal shift makes the first Cholesky safe up to
// cond ~ 1/u; two more passes restore orthogonality).  CholeskyQR2:
//   G = S^H S = R1^H R1,  Q1 = S R1^{-1},  Q1^H Q1 = R2^H R2,  R = R2 R1.
// Two Gram passes on tensor-core ZHERK instead of Householder panels (~3x
// fewer cycles at the BASELINE shapes).  R equals Householder's R up to a
// unitary diagonal D (R_hh = D R), which leaves every downstream quantity
// unchanged: z = Q R^{-H} b with Q = Q1 R2^{-1}, and CG on A^H R'^{-1} is invariant under
// R' -> D R' (the iterates rotate, their norms do not).  Stable while
// eps * cond(S)^2 < 1; returns false (caller falls back to Householder, as
// the reference) when a Cholesky breaks down or Q1 = S R1^{-1} is not orthonormal
// to 1e-3 (cond(S) above ~2e6).  On success ctx.qwork holds Q1 and ctx.R2 holds R2.
// r1_only: stop after the first Cholesky (R = R1, ctx.gram holds it too) -- Step 2's
// corrected seminormal solve (step2_z_csne) needs nothing more.
// One record per sketch QR on the device (and its pinned mirror): what the Cholesky, the inverse
// and the refinement kernels found, read by the host once.
struct QrStatus {
    CholStatus chol;
    RefineStatus ref;
    CholStatus chol1;  // shifted two-pass chain: the first (shifted) pass; `chol` is then the second
};
QrStatus* qr_status_dev(Context& ctx) { return dev<QrStatus>(ctx.qr_status, 1); }
const QrStatus& read_qr_status(Context& ctx) {
    auto* h = static_cast<QrStatus*>(ctx.pin_qr.ensure(sizeof(QrStatus)));
    MNB_CUDA(cudaMemcpyAsync(h, qr_status_dev(ctx), sizeof(QrStatus), cudaMemcpyDeviceToHost, ctx.stream));
    MNB_CUDA(cudaStreamSynchronize(ctx.stream));
    return *h;
}
// seeded dense start vector of the preconditioner check's power steps (splitmix64), uploaded
// through page-locked staging (no stream synchronization): device pointer (ctx.vec_m[11])
void power_start_vector(std::vector<double2>& v0, int64_t m);
double2* upload_power_start(Context& ctx, int64_t m) {
    std::vector<double2> v0;
    power_start_vector(v0, m);
    double2* vp = static_cast<double2*>(ctx.pin_vec.ensure(size_t(2 * m) * 16)) + m;
    std::memcpy(vp, v0.data(), size_t(m) * 16);
    double2* vstart = dev<double2>(ctx.vec_m[11], size_t(m));
    MNB_CUDA(cudaMemcpyAsync(vstart, vp, size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
    return vstart;
}
void power_start_vector(std::vector<double2>& v0, int64_t m) {
    v0.resize(size_t(m));
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (int64_t i = 0; i < m; ++i) {
        auto nxt = [&h] {
            uint64_t z = (h += 0x9E3779B97F4A7C15ull);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            return double((z ^ (z >> 31)) >> 11) * 0x1.0p-53 - 0.5;
        };
        v0[size_t(i)] = make_double2(nxt(), nxt());
    }
}
// scratch of launch_sketch_refine: three m-vectors, the ||z||^2 partials
void refine_scratch(Context& ctx, RefineArgs& a) {
    a.v0 = dev<double2>(ctx.vec_m[8], size_t(a.m));
    a.v1 = dev<double2>(ctx.vec_m[9], size_t(a.m));
    a.v2 = dev<double2>(ctx.vec_m[10], size_t(a.m));
    a.part = dev<double>(ctx.qr_part, size_t(a.l / 32 + 64));
}

// Shifted two-pass CholeskyQR for sketches with u cond(S)^2 not small (BASELINE c3, kappa = 1e8),
// queued on ctx.stream without a host round trip:
//   R1 = chol(G + s I)  (s = 11 (l m + m (m + 1)) u trace(G), Fukaya et al.),  X1 = R1^{-1},
//   Q1 = S X1,  R2 = chol(Q1^H Q1),  X2 = R2^{-1},  X = X1 X2 = (R2 R1)^{-1}.
// The shift caps cond(Q1) near sqrt(||S||^2 / s) ~ 1e4, so Q2 = Q1 X2 = S X is orthonormal to
// ~u cond(Q1)^2 ~ 1e-8: enough for the CG preconditioner (1e-3 is, lsq.cpp:66-69), and a
// contraction factor of 1e-8 for Step 2's corrected seminormal equations -- the third pass of
// shifted CholeskyQR3 (which buys R itself to O(u)) is not needed by either.  The Gram products
// and Q1 = S X1, X = X1 X2 are cuBLAS level-3 calls; the factorizations, inverses and the checks
// behind them are k_cholqr.cu's.  G0: S^H S on entry (overwritten by R1).  Records: qs->chol1
// (pass 1, its `deficient` = the rank rule on diag(R2 R1)), qs->chol (pass 2).
struct ShiftedChain {
    double2* Q1;  // l x m (ctx.qwork)
    double2* X2;  // m x m (ctx.R2)
    double2* X;   // m x m (ctx.Rinv)
};
ShiftedChain launch_shifted_chain(Context& ctx, const double2* S, int64_t l, int64_t m, double2* G0, double rank_rows,
                                  DevTrace* dt) {
    QrStatus* qs = qr_status_dev(ctx);
    double2* G2 = dev<double2>(ctx.gram, size_t(m) * size_t(m));
    double2* X1 = dev<double2>(ctx.tri_x1, size_t(m) * size_t(m));
    ShiftedChain c;
    c.Q1 = dev<double2>(ctx.qwork, size_t(l) * size_t(m));
    c.X2 = dev<double2>(ctx.R2, size_t(m) * size_t(m));
    c.X = dev<double2>(ctx.Rinv, size_t(m) * size_t(m));
    double2* W = dev<double2>(ctx.tri_work, size_t(m) * size_t(m));
    const double shift_factor = 11.0 * (double(l) * double(m) + double(m) * double(m + 1)) * kEps;
    const cuDoubleComplex cone = make_cuDoubleComplex(1.0, 0.0);
    const double one = 1.0, zero = 0.0;
    launch_chol_upper(G0, m, m, shift_factor, 0.0, &qs->chol1, ctx.num_sms, ctx.stream);
    if (dt) dt->mark("chol(G + sI)");
    launch_trtri_upper(G0, m, m, X1, W, &qs->chol1, ctx.num_sms, ctx.stream, true);
    if (dt) dt->mark("X1");
    cublas_check(cublasZtrmm(ctx.cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                             int(l), int(m), &cone, reinterpret_cast<const cuDoubleComplex*>(X1), int(m),
                             reinterpret_cast<const cuDoubleComplex*>(S), int(l),
                             reinterpret_cast<cuDoubleComplex*>(c.Q1), int(l)),
                 "ztrmm (Q1 = S X1)");
    if (dt) dt->mark("Q1 = S X1");
    cublas_check(cublasZherk(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, int(m), int(l), &one,
                             reinterpret_cast<const cuDoubleComplex*>(c.Q1), int(l), &zero,
                             reinterpret_cast<cuDoubleComplex*>(G2), int(m)),
                 "zherk");
    if (dt) dt->mark("gram");
    launch_chol_upper(G2, m, m, 0.0, 0.0, &qs->chol, ctx.num_sms, ctx.stream);
    if (dt) dt->mark("chol");
    launch_trtri_upper(G2, m, m, c.X2, W, &qs->chol, ctx.num_sms, ctx.stream, true);
    if (dt) dt->mark("X2");
    cublas_check(cublasZtrmm(ctx.cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                             int(m), int(m), &cone, reinterpret_cast<const cuDoubleComplex*>(c.X2), int(m),
                             reinterpret_cast<const cuDoubleComplex*>(X1), int(m),
                             reinterpret_cast<cuDoubleComplex*>(c.X), int(m)),
                 "ztrmm (X = X1 X2)");
    if (rank_rows > 0.0) launch_diag_product_rank(G2, m, G0, m, m, rank_rows, &qs->chol1, ctx.stream);
    if (dt) dt->mark("X = X1 X2");
    ctx.launches += 5;
    return c;
}
// the verdict of a shifted chain from its two Cholesky records
bool shifted_chain_ok(const QrStatus& h) {
    auto usable = [](const CholStatus& c) {
        if (c.info != 0 || !(c.dmin > 0.0)) return false;
        const double r = c.dmax / c.dmin;
        return !(kEps * r * r > 1e-3);
    };
    return usable(h.chol1) && usable(h.chol);
}

bool cholqr_r(Context& ctx, const double2* S, int64_t l, int64_t m, double2* R, bool shifted, bool* precond_only,
              bool r1_only = false, double rank_rows = 0.0, int64_t* deficient = nullptr) {
    double2* G = dev<double2>(ctx.gram, size_t(m) * size_t(m));
    double2* Q = dev<double2>(ctx.qwork, size_t(l) * size_t(m));
    double2* Rp = dev<double2>(ctx.R2, size_t(m) * size_t(m));
    int* info = dev<int>(ctx.qr_info, 2);
    QrStatus* qs = qr_status_dev(ctx);
    std::vector<double> diag(size_t(2 * m));
    int info_h = 0;
    double dmin_h = 0.0, dmax_h = 0.0;
    if (deficient) *deficient = -1;
    const double one = 1.0, zero = 0.0;
    const cuDoubleComplex cone = make_cuDoubleComplex(1.0, 0.0);
    auto herk = [&](const double2* X, double2* out) {
        cublas_check(cublasZherk(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, int(m), int(l), &one,
                                 reinterpret_cast<const cuDoubleComplex*>(X), int(l), &zero,
                                 reinterpret_cast<cuDoubleComplex*>(out), int(m)),
                     "zherk");
    };
    auto read_diag = [&](const double2* A) {
        MNB_CUDA(cudaMemcpy2DAsync(diag.data(), 16, A, size_t(m + 1) * 16, 16, size_t(m), cudaMemcpyDeviceToHost,
                                   ctx.stream));
        MNB_CUDA(cudaStreamSynchronize(ctx.stream));
    };
    // Upper Cholesky in place (+ a diagonal shift shift_factor * trace): the hand-written blocked
    // kernel and one status read, or (MNB_QR_LIB=1) cuSOLVER Xpotrf steered from the host
    auto potrf = [&](double2* A, double shift_factor) {
        if (!ctx.qr_lib) {
            launch_chol_upper(A, m, m, shift_factor, rank_rows, &qs->chol, ctx.num_sms, ctx.stream);
            ctx.launches += 1;
            const QrStatus& h = read_qr_status(ctx);
            info_h = h.chol.info;
            dmin_h = h.chol.dmin;
            dmax_h = h.chol.dmax;
            if (deficient && info_h == 0 && rank_rows > 0.0) *deficient = h.chol.deficient;
            return;
        }
        if (shift_factor > 0.0) {
            read_diag(A);
            double tr = 0.0;
            for (int64_t j = 0; j < m; ++j) tr += diag[size_t(2 * j)];
            launch_add_diagonal(A, m, shift_factor * tr, ctx.stream);
            ctx.launches += 1;
        }
        size_t dws = 0, hws = 0;
        cusolver_check(cusolverDnXpotrf_bufferSize(ctx.cusolver, ctx.cusolver_params, CUBLAS_FILL_MODE_UPPER, m,
                                                   CUDA_C_64F, A, m, CUDA_C_64F, &dws, &hws),
                       "potrf_bufferSize");
        void* work = ctx.qr_work.ensure(std::max<size_t>(dws, 16));
        if (ctx.host_work.size() < hws + 16) ctx.host_work.resize(hws + 16);
        cusolver_check(cusolverDnXpotrf(ctx.cusolver, ctx.cusolver_params, CUBLAS_FILL_MODE_UPPER, m, CUDA_C_64F, A, m,
                                        CUDA_C_64F, work, dws, ctx.host_work.data(), hws, info),
                       "potrf");
        launch_zero_lower(A, m, ctx.stream);
        ctx.launches += 1;
        MNB_CUDA(cudaMemcpyAsync(&info_h, info, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
        read_diag(A);
        dmax_h = 0.0;
        dmin_h = 1e300;
        for (int64_t j = 0; j < m; ++j) {
            const double a = std::hypot(diag[size_t(2 * j)], diag[size_t(2 * j + 1)]);
            dmax_h = std::max(dmax_h, a);
            dmin_h = std::min(dmin_h, a);
        }
    };
    auto trsm_q = [&](const double2* Rt) {  // Q <- Q Rt^{-1}
        cublas_check(cublasZtrsm(ctx.cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                                 CUBLAS_DIAG_NON_UNIT, int(l), int(m), &cone,
                                 reinterpret_cast<const cuDoubleComplex*>(Rt), int(m),
                                 reinterpret_cast<cuDoubleComplex*>(Q), int(l)),
                     "ztrsm");
    };
    // the diagonal ratio of R1 bounds cond(S) from below: once u ratio^2 > 1e-3 neither a second
    // Cholesky pass nor the seminormal corrections can reach orthogonality / the rounding floor
    // (c3, kappa = 1e8): hand over to shifted CholeskyQR3 at once instead of failing later
    auto ratio_bad = [&] { return !(dmin_h > 0.0) || kEps * (dmax_h / dmin_h) * (dmax_h / dmin_h) > 1e-3; };
    DevTrace dt(ctx, shifted ? "cholqr (shifted)" : "cholqr");
    struct DumpAtExit {
        DevTrace& d;
        ~DumpAtExit() {
            try {
                d.dump();
            } catch (...) {
            }
        }
    } dump_at_exit{dt};
    // pass 1: G = S^H S (+ shift) = R1^H R1, Q1 = S R1^{-1}  (or the Gram built during the sketch)
    if (ctx.pre_gram && !shifted)
        MNB_CUDA(cudaMemcpyAsync(G, ctx.pre_gram, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
    else
        herk(S, G);
    dt.mark("gram");
    // shifted CholeskyQR (Fukaya et al.): s = 11 (l m + m (m + 1)) u ||S||^2, ||S||_2^2 <= trace(G)
    const double shift_factor = shifted ? 11.0 * (double(l) * double(m) + double(m) * double(m + 1)) * kEps : 0.0;
    const bool fast_precond = !ctx.qr_lib && ctx.fastqr && !shifted && precond_only && *precond_only;
    if (fast_precond) {
        // The CG preconditioner needs only an R1 with Q1 = E R1^{-1} near-orthonormal (the CG rate and
        // its stopping bound sigma_min(B R'^{-1}) >= 1, lsq.cpp:66-69, then move by < 1e-3): Cholesky,
        // R1^{-1} (which the CG forms anyway, left in ctx.Rinv) and the check of ||Q1^H Q1 - I|| are
        // three launches queued back to back; the host reads their verdict once.
        double2* Rinv = dev<double2>(ctx.Rinv, size_t(m) * size_t(m));
        // (the Gram is kept in R: if this pass turns out unusable the shifted chain restarts from it)
        MNB_CUDA(cudaMemcpyAsync(R, G, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
        ctx.gram0 = R;
        launch_chol_upper(G, m, m, 0.0, rank_rows, &qs->chol, ctx.num_sms, ctx.stream);
        dt.mark("chol");
        upper_inverse(ctx, G, m, m, Rinv, &qs->chol);
        dt.mark("inverse");
        RefineArgs ra;
        ra.mode = REFINE_PRECOND;
        ra.S = S;
        ra.l = l;
        ra.m = m;
        ra.X = Rinv;
        ra.chol = &qs->chol;
        ra.b = upload_power_start(ctx, m);
        ra.z = dev<double2>(ctx.qprobe, size_t(l));
        refine_scratch(ctx, ra);
        ra.st = &qs->ref;
        ra.two_norm_check = ctx.two_norm_check ? 1 : 0;
        launch_sketch_refine(ra, ctx.num_sms, ctx.stream);
        dt.mark("check");
        ctx.launches += 2;
        const QrStatus& h = read_qr_status(ctx);
        trace("  cholqr: gram + chol + R1^-1 + check (one read)");
        info_h = h.chol.info;
        dmin_h = h.chol.dmin;
        dmax_h = h.chol.dmax;
        if (info_h != 0 || ratio_bad()) return false;
        if (deficient && rank_rows > 0.0) *deficient = h.chol.deficient;
        if (std::getenv("MNB_TRACE"))
            std::fprintf(stderr, "[mnb] one-pass preconditioner: u cond^2 <= %.2e (Frobenius), ||Q1^H Q1 - I|| ~ %.2e (%d steps)\n",
                         h.ref.thr, h.ref.best, h.ref.iterations);
        if (h.ref.accepted) {
            ctx.gram0 = nullptr;
            MNB_CUDA(cudaMemcpyAsync(R, G, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
            return true;
        }
        ctx.gram0 = nullptr;    // (R receives R1 below)
        *precond_only = false;  // R'^{-1} in ctx.Rinv is stale: the full factorization follows from R1
    } else {
        potrf(G, shift_factor);
        dt.mark("chol");
        trace("  cholqr: gram + potrf");
        if (info_h != 0) return false;
        if (!shifted && ratio_bad()) return false;
    }
    if (r1_only) {
        MNB_CUDA(cudaMemcpyAsync(R, G, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
        return true;
    }
    if (precond_only && *precond_only) {
        // (MNB_FASTQR=0 / MNB_QR_LIB=1: the same acceptance steered from the host)  The bound
        // |Q1^H Q1 - I| ~ u cond(E)^2 <= u ||R1||_F^2 ||R1^{-1}||_F^2 first.
        double2* Rinv = dev<double2>(ctx.Rinv, size_t(m) * size_t(m));
        upper_inverse(ctx, G, m, m, Rinv);
        double nr = 0.0, nri = 0.0;  // lower triangles are zero
        cublas_check(cublasDznrm2(ctx.cublas, int(m * m), reinterpret_cast<const cuDoubleComplex*>(G), 1, &nr), "dznrm2");
        cublas_check(cublasDznrm2(ctx.cublas, int(m * m), reinterpret_cast<const cuDoubleComplex*>(Rinv), 1, &nri),
                     "dznrm2");
        // The Frobenius norms overestimate the 2-norms by up to sqrt(m) each (~150 each for the
        // log-spaced spectra of the BASELINE configs).  When they alone reject, measure the loss
        // of orthogonality itself: ten power steps on the Hermitian D = Q1^H Q1 - I with
        // Q1 = E R1^{-1} (two GEMVs over E and two triangular products per step, from a seeded
        // dense start); ||D v|| for the unit v bounds ||D||_2 from below, so a factor-2 margin is
        // applied (accept on 2 ||D v|| <= 1e-3; c5: ~1e-4).
        trace("  cholqr: R1^-1 + Frobenius");
        bool accept = kEps * nr * nr * nri * nri <= 1e-3;
        if (!accept && ctx.two_norm_check) {
            double2* v = dev<double2>(ctx.vec_m[8], size_t(m));
            double2* a = dev<double2>(ctx.vec_m[9], size_t(m));
            double2* q = dev<double2>(ctx.qprobe, size_t(l));
            auto* vc = reinterpret_cast<cuDoubleComplex*>(v);
            auto* ac = reinterpret_cast<cuDoubleComplex*>(a);
            auto* qc = reinterpret_cast<cuDoubleComplex*>(q);
            const auto* Sc = reinterpret_cast<const cuDoubleComplex*>(S);
            const auto* Ri = reinterpret_cast<const cuDoubleComplex*>(Rinv);
            const cuDoubleComplex czero = make_cuDoubleComplex(0.0, 0.0);
            std::vector<double2> v0;
            power_start_vector(v0, m);
            MNB_CUDA(cudaMemcpyAsync(v, v0.data(), size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
            // device pointer mode: the ten steps run without a host round trip; one read at the end
            double* nrm_d = dev<double>(ctx.scratch, 512);
            cublasSetPointerMode(ctx.cublas, CUBLAS_POINTER_MODE_DEVICE);
            cuDoubleComplex* consts = reinterpret_cast<cuDoubleComplex*>(nrm_d + 8);  // [1, 0]
            const cuDoubleComplex hc[2] = {cone, czero};
            MNB_CUDA(cudaMemcpyAsync(consts, hc, sizeof hc, cudaMemcpyHostToDevice, ctx.stream));
            cublas_check(cublasDznrm2(ctx.cublas, int(m), vc, 1, nrm_d), "dznrm2");
            for (int it = 0; it < 10; ++it) {
                launch_unit_copy(v, a, m, nrm_d, ctx.stream);                    // v = v / ||v||, a = v
                // (R1^{-1}: its strict lower triangle is exactly zero, so a plain
                // GEMV -- one streaming read, no triangular dependency chain -- applies it)
                cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_N, int(m), int(m), consts, Ri, int(m), vc, 1, consts + 1,
                                         ac, 1), "zgemv");                      // a = R1^{-1} v
                cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_N, int(l), int(m), consts, Sc, int(l), ac, 1, consts + 1,
                                         qc, 1), "zgemv");                      // q = E a
                cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_C, int(l), int(m), consts, Sc, int(l), qc, 1, consts + 1,
                                         ac, 1), "zgemv");                      // a = E^H q
                cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_C, int(m), int(m), consts, Ri, int(m), ac, 1, consts + 1,
                                         qc, 1), "zgemv");                      // q = R1^{-H} a
                launch_sub_copy(qc, v, m, ctx.stream);                           // v = q - v = D v
                cublas_check(cublasDznrm2(ctx.cublas, int(m), vc, 1, nrm_d), "dznrm2");  // ||D v||
                ctx.launches += 2;
            }
            cublasSetPointerMode(ctx.cublas, CUBLAS_POINTER_MODE_HOST);
            double lam = 0.0;
            MNB_CUDA(cudaMemcpyAsync(&lam, nrm_d, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
            MNB_CUDA(cudaStreamSynchronize(ctx.stream));
            trace("  cholqr: ||Q1^H Q1 - I|| power steps");
            accept = 2.0 * lam <= 1e-3;
            if (std::getenv("MNB_TRACE"))
                std::fprintf(stderr, "[mnb] one-pass preconditioner: u cond^2 <= %.2e (Frobenius), ||Q1^H Q1 - I|| ~ %.2e\n",
                             kEps * nr * nr * nri * nri, lam);
        }
        if (accept) {
            MNB_CUDA(cudaMemcpyAsync(R, G, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
            return true;
        }
        *precond_only = false;  // R'^{-1} in ctx.Rinv is stale: the full factorization follows
    }
    MNB_CUDA(cudaMemcpyAsync(Q, S, size_t(l) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
    trsm_q(G);
    MNB_CUDA(cudaMemcpyAsync(R, G, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
    dt.mark("Q1 = S R1^-1");
    // passes 2 (and 3): R_p = chol(Q^H Q); R <- R_p R; on the last pass Q must already be
    // orthonormal to 1e-3 (|Q^H Q - I| ~ eps cond^2) for R to be accurate -- else Householder.
    const int passes = shifted ? 3 : 2;
    for (int p = 2; p <= passes; ++p) {
        herk(Q, Rp);
        dt.mark("gram");
        if (p == passes) {
            double* dev_max = dev<double>(ctx.scratch, 512);
            launch_max_offset_from_identity(Rp, m, dev_max, ctx.stream);
            ctx.launches += 1;
            double gmax = 0.0;
            MNB_CUDA(cudaMemcpyAsync(&gmax, dev_max, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
            MNB_CUDA(cudaStreamSynchronize(ctx.stream));
            if (!(gmax < 1e-3)) return false;
        }
        potrf(Rp, 0.0);
        dt.mark("chol");
        if (info_h != 0) return false;
        if (p < passes) {
            trsm_q(Rp);
            dt.mark("Q = Q Rp^-1");
        }
        cublas_check(cublasZtrmm(ctx.cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                                 CUBLAS_DIAG_NON_UNIT, int(m), int(m), &cone, reinterpret_cast<const cuDoubleComplex*>(Rp),
                                 int(m), reinterpret_cast<const cuDoubleComplex*>(R), int(m),
                                 reinterpret_cast<cuDoubleComplex*>(R), int(m)),
                     "ztrmm");
        dt.mark("R = Rp R");
    }
    if (deficient) *deficient = -1;  // the rank rule applies to the final R: the caller reads its diagonal
    return true;  // ctx.qwork holds Q_{passes-1}, ctx.R2 the last R_p:  Q = Q_{passes-1} R_p^{-1}
}

// QR of a finished l x m sketch on ctx.stream (CholeskyQR2, else Householder); qr_s += device time.
// precond: the preconditioner's QR (E), which may stop after one Cholesky pass (path 3).
// seminormal: Step 2's QR (S), which may stop after R1 = chol(S^H S) (path 4) -- step2_z_csne
// then solves with the corrected seminormal equations and falls back here if they do not converge.
// rank_rows: the `rows` of the rank rule the caller will apply (lets the Cholesky kernel take it).
SketchQr qr_of_sketch(Context& ctx, double2* S, int64_t l, DevBuf& taubuf, DevBuf& Rbuf, double* qr_s,
                      bool precond = false, bool seminormal = false, double rank_rows = 0.0) {
    const int64_t m = ctx.m;
    double2* tau = dev<double2>(taubuf, size_t(m));
    double2* R = dev<double2>(Rbuf, size_t(m) * size_t(m));
    cudaEvent_t e1 = ctx.timer_event(), e2 = ctx.timer_event();
    MNB_CUDA(cudaEventRecord(e1, ctx.stream));
    SketchQr out{S, tau, R, m, false};
    out.path = 0;
    ctx.gram0 = nullptr;
    // CholeskyQR2; if the sketch is too ill-conditioned, shifted CholeskyQR3 (and once a sketch of
    // this solve needed it, the next one starts there); Householder (the reference's) as the last resort
    bool done = false;
    if (ctx.cholqr && seminormal && ctx.csne && !ctx.qr_shifted) {
        done = cholqr_r(ctx, S, l, m, R, false, nullptr, /*r1_only=*/true, rank_rows, &out.deficient);
        if (done) out.path = 4;
        else ctx.qr_shifted = true;  // the first Cholesky pass failed: CholeskyQR2 would too
    }
    if (ctx.cholqr && !done) {
        if (!ctx.qr_shifted) {
            bool one_pass = precond;
            done = cholqr_r(ctx, S, l, m, R, false, &one_pass, false, rank_rows, &out.deficient);
            if (done && one_pass) {
                out.path = 3;
                out.rinv_ready = true;
            }
            if (!done) ctx.qr_shifted = true;
        }
        if (!done && precond && ctx.fastqr && !ctx.qr_lib) {
            // the preconditioner of an ill-conditioned sketch: shifted two-pass chain + the check of
            // ||Q2^H Q2 - I|| on (Q1, X2), one host read (path 5)
            DevTrace dt(ctx, "shifted chain (E)");
            if (!ctx.gram0) {
                if (ctx.pre_gram)
                    MNB_CUDA(cudaMemcpyAsync(R, ctx.pre_gram, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice,
                                             ctx.stream));
                else {
                    const double one = 1.0, zero = 0.0;
                    cublas_check(cublasZherk(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, int(m), int(l), &one,
                                             reinterpret_cast<const cuDoubleComplex*>(S), int(l), &zero,
                                             reinterpret_cast<cuDoubleComplex*>(R), int(m)),
                                 "zherk");
                }
                dt.mark("gram");
            }
            ctx.gram0 = nullptr;
            const ShiftedChain ch = launch_shifted_chain(ctx, S, l, m, R, rank_rows, &dt);
            QrStatus* qs = qr_status_dev(ctx);
            RefineArgs ra;
            ra.mode = REFINE_PRECOND;
            ra.S = ch.Q1;
            ra.l = l;
            ra.m = m;
            ra.X = ch.X2;
            ra.chol = &qs->chol;
            ra.b = upload_power_start(ctx, m);
            ra.z = dev<double2>(ctx.qprobe, size_t(l));
            refine_scratch(ctx, ra);
            ra.st = &qs->ref;
            ra.two_norm_check = 1;
            launch_sketch_refine(ra, ctx.num_sms, ctx.stream);
            dt.mark("check");
            ctx.launches += 1;
            const QrStatus h = read_qr_status(ctx);
            dt.dump();
            if (std::getenv("MNB_TRACE"))
                std::fprintf(stderr, "[mnb] shifted chain (E): info %d/%d, diag ratios %.2e/%.2e, ||Q2^H Q2 - I|| ~ %.2e (%d steps, Frobenius bound %.2e) -> %s\n",
                             h.chol1.info, h.chol.info, h.chol1.dmax / h.chol1.dmin, h.chol.dmax / h.chol.dmin,
                             h.ref.best, h.ref.iterations, h.ref.thr,
                             shifted_chain_ok(h) && h.ref.accepted ? "accepted" : "fallback");
            if (shifted_chain_ok(h) && h.ref.accepted) {
                done = true;
                out.path = 5;
                out.rinv_ready = true;
                out.deficient = rank_rows > 0.0 ? h.chol1.deficient : -1;
            }
        }
        ctx.gram0 = nullptr;
        if (!done) {
            done = cholqr_r(ctx, S, l, m, R, true, nullptr);
            out.path = 1;
        }
    }
    if (!done) {
        qr_in_place(ctx, S, l, m, tau);
        out.R = S;
        out.ldR = l;
        out.householder = true;
        out.path = 2;
    }
    MNB_CUDA(cudaEventRecord(e2, ctx.stream));
    MNB_CUDA(cudaEventSynchronize(e2));
    float b = 0.f;
    MNB_CUDA(cudaEventElapsedTime(&b, e1, e2));
    if (qr_s) *qr_s += b * 1e-3;
    return out;
}

SketchQr sketch_and_qr(Context& ctx, const SrftDev& op, DevBuf& Sbuf, DevBuf& taubuf, DevBuf& Rbuf, double* kernel_ms,
                       double* sketch_s, double* qr_s, double* redistribute_s, bool precond = false) {
    const int64_t l = op.host->l, m = ctx.m;
    double2* S = dev<double2>(Sbuf, size_t(l) * size_t(m));
    cudaEvent_t e0 = ctx.timer_event(), e1 = ctx.timer_event();
    MNB_CUDA(cudaEventRecord(e0, ctx.stream));
    sketch_matrix(ctx, op, S, kernel_ms, redistribute_s);
    MNB_CUDA(cudaEventRecord(e1, ctx.stream));
    SketchQr out = qr_of_sketch(ctx, S, l, taubuf, Rbuf, qr_s, precond);
    float a = 0.f;
    MNB_CUDA(cudaEventElapsedTime(&a, e0, e1));
    if (sketch_s) *sketch_s += a * 1e-3;
    return out;
}

// Run a block of the solve on another stream: ctx.stream and the library handles follow.
struct OnStream {
    Context& c;
    cudaStream_t saved;
    OnStream(Context& ctx, cudaStream_t s) : c(ctx), saved(ctx.stream) { bind(s); }
    ~OnStream() { bind(saved); }
    void bind(cudaStream_t s) {
        c.stream = s;
        cublasSetStream(c.cublas, s);
        cusolverDnSetStream(c.cusolver, s);
    }
};

unsigned char* pinned_alloc(PinnedBuf& pb, size_t bytes) { return static_cast<unsigned char*>(pb.ensure(bytes)); }

void validate_matrix_set(const Context& ctx) {
    require(ctx.A != nullptr || ctx.n_local == 0, MNB_ERR_INVALID_ARGUMENT, "no problem matrix set (mnb_set_matrix)");
}

// Step 2 (src/solver.cpp:93-96): z = Q [R^{-H} b; 0] on ctx.stream.
void step2_z(Context& ctx, const SketchQr& sq, const double2* b_host, int64_t l, int64_t m, double2* z) {
    const auto* Rc = reinterpret_cast<const cuDoubleComplex*>(sq.R);
    if (sq.householder) {
        MNB_CUDA(cudaMemsetAsync(z, 0, size_t(l) * 16, ctx.stream));
        MNB_CUDA(cudaMemcpyAsync(z, b_host, size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
        cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, int(m), Rc,
                                 int(sq.ldR), reinterpret_cast<cuDoubleComplex*>(z), 1),
                     "ztrsv");
        int lwork = 0;
        cusolver_check(cusolverDnZunmqr_bufferSize(ctx.cusolver, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, int(l), 1, int(m),
                                                   reinterpret_cast<const cuDoubleComplex*>(sq.S), int(l),
                                                   reinterpret_cast<const cuDoubleComplex*>(sq.tau),
                                                   reinterpret_cast<const cuDoubleComplex*>(z), int(l), &lwork),
                       "unmqr_bufferSize");
        auto* work = static_cast<cuDoubleComplex*>(ctx.qr_work.ensure(size_t(std::max(lwork, 1)) * 16));
        cusolver_check(cusolverDnZunmqr(ctx.cusolver, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, int(l), 1, int(m),
                                        reinterpret_cast<const cuDoubleComplex*>(sq.S), int(l),
                                        reinterpret_cast<const cuDoubleComplex*>(sq.tau),
                                        reinterpret_cast<cuDoubleComplex*>(z), int(l), work, lwork,
                                        dev<int>(ctx.qr_info, 1)),
                       "unmqr");
        return;
    }
    // CholeskyQR2: Q = S R^{-1} = Q1 R2^{-1}, so z = Q1 (R2^{-1} (R^{-H} b))
    double2* w = dev<double2>(ctx.vec_m[6], size_t(m));
    MNB_CUDA(cudaMemcpyAsync(w, b_host, size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
    cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, int(m), Rc,
                             int(sq.ldR), reinterpret_cast<cuDoubleComplex*>(w), 1),
                 "ztrsv");
    cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, int(m),
                             reinterpret_cast<const cuDoubleComplex*>(ctx.R2.p), int(m),
                             reinterpret_cast<cuDoubleComplex*>(w), 1),
                 "ztrsv");
    const cuDoubleComplex cone = make_cuDoubleComplex(1.0, 0.0), czero = make_cuDoubleComplex(0.0, 0.0);
    cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_N, int(l), int(m), &cone,
                             reinterpret_cast<const cuDoubleComplex*>(ctx.qwork.p), int(l),
                             reinterpret_cast<const cuDoubleComplex*>(w), 1, &czero, reinterpret_cast<cuDoubleComplex*>(z),
                             1),
                 "zgemv");
}

// Step 2 on the first Cholesky factor only (path 4): z is the minimal-norm solution of
// S^H z = b (z = Q R^{-H} b = S (S^H S)^{-1} b, src/solver.cpp:93-96), from the corrected
// seminormal equations  z_0 = S G^{-1} b,  z_{k+1} = z_k + S G^{-1} (b - S^H z_k),  G = R1^H R1.
// Every iterate lies in range(S); the refinement is accepted once the residual is at the
// rounding level of S^H z (||b - S^H z|| <= 2 sqrt(l) u ||S||_F ||z||), which makes z as
// accurate as the Householder solve (error ~ u cond(S)).  Returns false (the caller runs the
// shifted CholeskyQR3 and step2_z) when a correction does not shrink the residual tenfold
// (u cond(S)^2 is not small) or three corrections do not get there.
bool step2_z_csne(Context& ctx, const SketchQr& sq, const double2* S, const double2* b_host, int64_t l, int64_t m,
                  double2* z) {
    const auto* R1 = reinterpret_cast<const cuDoubleComplex*>(sq.R);
    auto* zc = reinterpret_cast<cuDoubleComplex*>(z);
    const auto* Sc = reinterpret_cast<const cuDoubleComplex*>(S);
    double2* bd = dev<double2>(ctx.vec_m[6], size_t(m));
    double2* w = dev<double2>(ctx.vec_m[8], size_t(m));
    auto* wc = reinterpret_cast<cuDoubleComplex*>(w);
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), mone = make_cuDoubleComplex(-1.0, 0.0),
                          zero = make_cuDoubleComplex(0.0, 0.0);
    MNB_CUDA(cudaMemcpyAsync(bd, b_host, size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
    auto solve_gram = [&]() {  // w <- G^{-1} w = R1^{-1} R1^{-H} w
        cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, int(m), R1,
                                 int(sq.ldR), wc, 1),
                     "ztrsv");
        cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, int(m), R1,
                                 int(sq.ldR), wc, 1),
                     "ztrsv");
    };
    // ||S||_F^2 = trace(S^H S): the diagonal of R1^H R1 is the column sums of |R1|^2
    double sf = 0.0;
    cublas_check(cublasDznrm2(ctx.cublas, int(m * sq.ldR), R1, 1, &sf), "dznrm2");  // lower triangle is zero
    MNB_CUDA(cudaMemcpyAsync(w, bd, size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
    solve_gram();
    cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_N, int(l), int(m), &one, Sc, int(l), wc, 1, &zero, zc, 1), "zgemv");
    // Corrections run until the residual stops halving (iterative refinement to its floor: the
    // first correction alone left ||b - S^H z|| ~10x above Householder's at c2 / c5, and the
    // CG carries that error into x amplified by cond(A): 2.1e-9 vs 4.7e-11 against the exact p,
    // profiles/r02/b/acc_c2.log).  The floor is accepted when it is at the rounding level
    // 2 sqrt(l) u ||S||_F ||z||; otherwise (u cond(S)^2 not small) the caller falls back.
    const double thr = 2.0 * std::sqrt(double(l)) * kEps * sf;
    double prev = 0.0, best = 0.0, nz_best = 0.0;
    for (int it = 0; it <= 6; ++it) {
        // w = b - S^H z
        MNB_CUDA(cudaMemcpyAsync(w, bd, size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
        cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_C, int(l), int(m), &mone, Sc, int(l), zc, 1, &one, wc, 1),
                     "zgemv");
        // both norms on the device, one host read per correction
        double* nrm_d = dev<double>(ctx.scratch, 512);
        cublasSetPointerMode(ctx.cublas, CUBLAS_POINTER_MODE_DEVICE);
        cublas_check(cublasDznrm2(ctx.cublas, int(m), wc, 1, nrm_d), "dznrm2");
        cublas_check(cublasDznrm2(ctx.cublas, int(l), zc, 1, nrm_d + 1), "dznrm2");
        cublasSetPointerMode(ctx.cublas, CUBLAS_POINTER_MODE_HOST);
        double nrz[2];
        MNB_CUDA(cudaMemcpyAsync(nrz, nrm_d, sizeof nrz, cudaMemcpyDeviceToHost, ctx.stream));
        MNB_CUDA(cudaStreamSynchronize(ctx.stream));
        const double nr = nrz[0], nz = nrz[1];
        if (std::getenv("MNB_TRACE")) std::fprintf(stderr, "[mnb] csne it %d: ||b - S^H z|| = %.3e (thr %.3e)\n", it, nr, thr * nz);
        if (it == 0 || nr < best) {
            best = nr;
            nz_best = nz;
        }
        if (nr == 0.0) return true;
        // stagnated: the last correction did not halve the residual (or the budget is spent)
        if ((it > 0 && !(nr < 0.5 * prev)) || it == 6) break;
        prev = nr;
        solve_gram();
        cublas_check(cublasZgemv(ctx.cublas, CUBLAS_OP_N, int(l), int(m), &one, Sc, int(l), wc, 1, &one, zc, 1), "zgemv");
    }
    return best <= thr * nz_best;
}

// QR(S) and Step 2 (src/solver.cpp:85-97) queued on ctx.stream without a host round trip:
// G = S^H S (cuBLAS ZHERK, a plain library GEMM), R1 = chol(G) with the rank rule taken on its
// diagonal, X = R1^{-1}, then the corrected seminormal equations of step2_z_csne as one
// persistent kernel; their findings land in the context's QrStatus record.
// early_verdict: the host reads the Cholesky's verdict before it queues the rest and returns
// false when the factor cannot be used (pivot failure, or u (max / min of diag R)^2 > 1e-3) --
// the caller then goes straight to the shifted chain instead of running the inverse, the
// corrections and T^* z on a factor it will discard.  Returns true when everything is queued.
bool launch_fast_step2(Context& ctx, const double2* S, int64_t l, int64_t m, const double2* b_host, double2* z,
                       DevTrace* dt = nullptr, double2* keep_gram = nullptr, bool early_verdict = false) {
    double2* G = dev<double2>(ctx.gram, size_t(m) * size_t(m));
    double2* X = dev<double2>(ctx.R2, size_t(m) * size_t(m));
    QrStatus* qs = qr_status_dev(ctx);
    const double one = 1.0, zero = 0.0;
    double2* bd = dev<double2>(ctx.vec_m[6], size_t(m));
    {
        // (through page-locked staging: an async copy from pageable memory would first synchronize
        // the stream, i.e. make the host wait for the Cholesky and the inverse before queueing on)
        double2* bp = static_cast<double2*>(ctx.pin_vec.ensure(size_t(2 * m) * 16));
        std::memcpy(bp, b_host, size_t(m) * 16);
        MNB_CUDA(cudaMemcpyAsync(bd, bp, size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
    }
    cublas_check(cublasZherk(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, int(m), int(l), &one,
                             reinterpret_cast<const cuDoubleComplex*>(S), int(l), &zero,
                             reinterpret_cast<cuDoubleComplex*>(G), int(m)),
                 "zherk");
    if (dt) dt->mark("gram");
    if (keep_gram)  // the shifted chain restarts from the Gram if this pass turns out unusable
        MNB_CUDA(cudaMemcpyAsync(keep_gram, G, size_t(m) * size_t(m) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
    launch_chol_upper(G, m, m, 0.0, double(l), &qs->chol, ctx.num_sms, ctx.stream);
    if (dt) dt->mark("chol");
    ctx.launches += 1;
    if (early_verdict) {
        const QrStatus& h = read_qr_status(ctx);
        const double ratio = h.chol.dmin > 0.0 ? h.chol.dmax / h.chol.dmin : 1e300;
        if (h.chol.info != 0 || kEps * ratio * ratio > 1e-3) return false;
    }
    upper_inverse(ctx, G, m, m, X, &qs->chol);
    if (dt) dt->mark("inverse");
    RefineArgs ra;
    ra.mode = REFINE_CSNE;
    ra.S = S;
    ra.l = l;
    ra.m = m;
    ra.X = X;
    ra.chol = &qs->chol;
    ra.b = bd;
    ra.z = z;
    refine_scratch(ctx, ra);
    ra.st = &qs->ref;
    launch_sketch_refine(ra, ctx.num_sms, ctx.stream);
    if (dt) dt->mark("csne");
    ctx.launches += 1;
    return true;
}

void csne_solve_host(Context& ctx, const double2* S, int64_t l, int64_t m, const double2* b, double2* z,
                     double* status) {
    double2* Sd = dev<double2>(ctx.sk_S, size_t(l) * size_t(m));
    double2* zd = dev<double2>(ctx.rhs, size_t(l));
    MNB_CUDA(cudaMemcpyAsync(Sd, S, size_t(l) * size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
    cublasSetStream(ctx.cublas, ctx.stream);
    launch_fast_step2(ctx, Sd, l, m, b, zd);
    const QrStatus h = read_qr_status(ctx);
    MNB_CUDA(cudaMemcpyAsync(z, zd, size_t(l) * 16, cudaMemcpyDeviceToHost, ctx.stream));
    sync(ctx);
    status[0] = (h.chol.info == 0 && h.ref.accepted) ? 1.0 : 0.0;
    status[1] = h.ref.iterations;
    status[2] = h.ref.best;
    status[3] = h.ref.nz_best;
}

// ---------------------------------------------------- solve_randomized ----
void solve_randomized(Context& ctx, const double2* b_host, const mnb_solver_config& cfg, double2* x_dev,
                      double2* c_dev, mnb_solve_report& rep) {
    const double t_start = now_s();
    ctx.timers.clear();  // drop timers of an aborted call (they point into its report)
    ctx.timer_next = 0;
    ctx.qr_shifted = false;
    ctx.init_from_sketch = false;
    validate_matrix_set(ctx);
    const int64_t m = ctx.m, n = ctx.n_global;
    // ProblemInstance::validate (src/solver.cpp:37-48); A's finiteness is checked on the device below.
    if (m < 1 || m >= n)
        throw Error(MNB_ERR_DIMENSION, "problem must be underdetermined: 1 <= m < n, got m=" + std::to_string(m) +
                                           ", n=" + std::to_string(n));
    bool b_finite = true, b_zero = true;
    for (int64_t i = 0; i < 2 * m; ++i) {
        const double v = reinterpret_cast<const double*>(b_host)[i];
        b_finite = b_finite && std::isfinite(v);
        b_zero = b_zero && v == 0.0;
    }
    if (!b_finite) throw Error(MNB_ERR_DIMENSION, "matrix and right-hand side entries must be finite");
    if (!(cfg.epsilon > 0.0 && cfg.epsilon < 1.0)) throw Error(MNB_ERR_CONFIG, "epsilon must lie in (0, 1)");
    if (!(cfg.alpha > 1.0)) throw Error(MNB_ERR_CONFIG, "alpha must exceed 1");
    const int64_t l = cfg.sketch_size > 0 ? cfg.sketch_size : 4 * m;
    if (l <= m || l >= n)
        throw Error(MNB_ERR_CONFIG, "sketch size l=" + std::to_string(l) + " must satisfy m < l < n (m=" +
                                        std::to_string(m) + ", n=" + std::to_string(n) +
                                        "); this system is outside the randomized solver's regime - use the "
                                        "classical solver instead");
    rep = mnb_solve_report{};
    rep.sketch_size = l;
    rep.lsq_tau = cfg.epsilon * cfg.epsilon * double(l) / (cfg.alpha * double(n));
    rep.world_size = ctx.world;
    rep.lsq_converged = 1;
    const int64_t launches0 = ctx.launches;
    // a deferred host copy never outlives this call (the caller may release its buffer on return)
    struct ResidentGuard {
        Context& c;
        ~ResidentGuard() {
            if (c.pending_host) {
                try {
                    c.make_resident();
                } catch (...) {
                }
            }
        }
    } resident_guard{ctx};
    if (b_zero) {  // src/solver.cpp:68-73
        if (ctx.n_local) {
            MNB_CUDA(cudaMemsetAsync(x_dev, 0, size_t(ctx.n_local) * 16, ctx.stream));
            if (c_dev) MNB_CUDA(cudaMemsetAsync(c_dev, 0, size_t(ctx.n_local) * 16, ctx.stream));
        }
        sync(ctx);
        rep.total_seconds = now_s() - t_start;
        return;
    }
    const int sampling = cfg.sampling;
    const RandomStream root(cfg.seed);
    const uint64_t seed_T = root.derive_seed(11), seed_Tp = root.derive_seed(12);  // src/solver.cpp:19
    // host threads for the parameter draws (MNB_HOST_THREADS overrides the core count)
    static const int hw = [] {
        const char* e = std::getenv("MNB_HOST_THREADS");
        const int v = e ? std::atoi(e) : 0;
        return v >= 2 ? v : int(std::max(2u, std::thread::hardware_concurrency()));
    }();
    // Deferred host A (MNB_HOST_ASYNC, one GPU): copy it in row slabs on a side stream now; both
    // sketches then run slab by slab as the rows land, so the H2D hides the parameter draws, the
    // sketches and most of Step 1.  Otherwise A is already resident.
    const bool pipelined = ctx.pending_host && !ctx.distributed() && ctx.n_local > 0;
    ctx.slab_ready = false;  // distributed: this solve's one all-to-all feeds both sketches
    std::vector<std::pair<int64_t, int64_t>> slabs;  // (row0, rows)
    if (!pipelined) ctx.make_resident();
    // T (needed first) is drawn with every host thread; T' is drawn in the background with half
    // of them while this thread drives Steps 1-3 on the GPU.  Pipelined: the first row slab of A
    // goes out first, both operators are drawn while it is in flight, their (small) uploads queue
    // behind it on the copy engine, then the remaining slabs follow.
    SrftHost T, Tp;
    auto noop = [](unsigned char*) {};
    double t_param_T = 0.0, t_param_Tp = 0.0;
    auto build_T = [&](int threads) {
        const double s = now_s();
        build_srft_host(T, l, n, seed_T, sampling, [&](size_t bytes) { return pinned_alloc(ctx.pin_params[0], bytes); },
                        noop, threads);
        t_param_T = now_s() - s;
    };
    auto build_Tp = [&](int threads) {
        const double s = now_s();
        build_srft_host(Tp, l, n, seed_Tp, sampling, [&](size_t bytes) { return pinned_alloc(ctx.pin_params[1], bytes); },
                        noop, threads);
        t_param_Tp = now_s() - s;
    };
    SrftStage stage_T;  // (before the join guards: the builder signals it)
    const double t_start_T = now_s();
    double t_first_T = 0.0;
    std::future<void> fut_Tp, fut_T;
    // host_async futures do not block on destruction: join the draw before T/T' go out of scope
    struct JoinGuard {
        std::future<void>& f;
        ~JoinGuard() { if (f.valid()) f.wait(); }
    } join_Tp{fut_Tp}, join_T_staged{fut_T};
    // Staged draw of T (A resident, n >= MNB_STAGED_MIN_N, default 2^16; MNB_STAGED_DRAW=0: off)
    static const int64_t staged_min_n = [] {
        if (const char* e = std::getenv("MNB_STAGED_DRAW"); e && std::atoi(e) == 0) return int64_t(1) << 62;
        const char* e = std::getenv("MNB_STAGED_MIN_N");
        const long long v = e ? std::atoll(e) : 0;
        return int64_t(v >= 2 ? v : 65536);
    }();
    const bool staged = !pipelined && n >= staged_min_n;
    struct StageHookGuard {  // the hook captures this frame
        Context& c;
        ~StageHookGuard() { c.after_first_stage = nullptr; }
    } stage_hook_guard{ctx};
    SrftDev& Td = ctx.op_dev[0];
    SrftDev& Tpd = ctx.op_dev[1];
    if (pipelined) {
        if (!ctx.copy_stream) MNB_CUDA(cudaStreamCreateWithFlags(&ctx.copy_stream, cudaStreamNonBlocking));
        // eight row slabs; only the last one's sketches are exposed after the copy, so it is the
        // short one (m / 32 rows, at least 64) and the other seven share the rest
        // (MNB_EVEN_SLABS=1: eight equal slabs)
        static const bool even_slabs = std::getenv("MNB_EVEN_SLABS") && std::atoi(std::getenv("MNB_EVEN_SLABS")) == 1;
        if (m >= 1024 && !even_slabs) {
            const int64_t body = (m - std::max<int64_t>(64, m / 32)) & ~int64_t(7);  // slab starts at multiples of 8
            const int64_t last = m - body;
            const int64_t per = ((body + 6) / 7 + 7) & ~int64_t(7);
            for (int64_t r0 = 0; r0 < body; r0 += per) slabs.emplace_back(r0, std::min(per, body - r0));
            slabs.emplace_back(body, last);
        } else {
            const int64_t per = std::max<int64_t>(64, ((m + 7) / 8 + 7) & ~int64_t(7));
            for (int64_t r0 = 0; r0 < m; r0 += per) slabs.emplace_back(r0, std::min(per, m - r0));
        }
        const size_t e = ctx.esz();
        auto issue = [&](size_t k) {
            const auto [r0, rows] = slabs[k];
            MNB_CUDA(cudaMemcpy2DAsync(static_cast<unsigned char*>(ctx.A_own.p) + size_t(r0) * e, size_t(m) * e,
                                       static_cast<const unsigned char*>(ctx.A_host) + size_t(r0) * e,
                                       size_t(ctx.host_lda) * e, size_t(rows) * e, size_t(ctx.n_local),
                                       cudaMemcpyHostToDevice, ctx.copy_stream));
            MNB_CUDA(cudaEventRecord(ctx.event(200 + k), ctx.copy_stream));
        };
        MNB_CUDA(cudaEventRecord(ctx.event(199), ctx.copy_stream));
        issue(0);
        const double tp0 = now_s();
        auto f1 = host_async([&] { build_T(std::max(1, hw / 2)); });
        JoinGuard join_T{f1};
        build_Tp(std::max(1, hw - hw / 2));
        f1.get();
        (void)tp0;
        // the operator uploads go on the copy stream between slab 0 and slab 1: the copy engine does
        // not keep issue order across streams, and uploads on the solve stream landed only after
        // every slab of A (the sketches then waited for the whole H2D)
        {
            const cudaStream_t solve_stream = ctx.stream;
            ctx.stream = ctx.copy_stream;
            upload_srft(ctx, T, Td);
            MNB_CUDA(cudaEventRecord(ctx.event(230), ctx.stream));
            upload_srft(ctx, Tp, Tpd);
            MNB_CUDA(cudaEventRecord(ctx.event(231), ctx.stream));
            ctx.stream = solve_stream;
            MNB_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.event(231), 0));
        }
        trace("uploads issued");
        for (size_t k = 1; k < slabs.size(); ++k) issue(k);
    } else if (staged) {
        // T's groups of the first H stage (perm~, theta~, zeta~, zeta) are drawn first; that stage
        // is queued as soon as they are uploaded, and the rest of T follows behind it (below)
        fut_T = host_async([&] {
            try {
                build_srft_host(T, l, n, seed_T, sampling,
                                [&](size_t bytes) { return pinned_alloc(ctx.pin_params[0], bytes); }, noop, hw, &stage_T);
            } catch (...) {
                stage_T.signal(2);
                throw;
            }
            t_param_T = now_s() - t_start_T;
        });
        fut_Tp = host_async([&] { build_Tp(std::max(1, hw / 2)); });
        if (!stage_T.wait_first()) fut_T.get();  // rethrows the builder's error
        t_first_T = now_s() - t_start_T;
    } else {
        build_T(hw);
        fut_Tp = host_async([&] { build_Tp(std::max(1, hw / 2)); });
    }

    // Streams: the sketches and the CG passes (memory-bound) run on ctx.stream; the QRs and
    // Steps 2-3 (tensor-core / latency-bound) run on an auxiliary stream beside them:
    //   s1: sketch S | sketch E | INIT pass (after c) | CG (after R')
    //   s2:          | QR(S), Step 2, Step 3 (c)      | QR(E)
    // Every NCCL call (all-to-all, allgathers, the finiteness allreduce, the CG allreduces) is
    // issued on s1 in the same host order on every rank; s2 carries none.
    trace("params done");
    cudaStream_t s1 = ctx.stream;
    if (!ctx.aux_stream) MNB_CUDA(cudaStreamCreateWithFlags(&ctx.aux_stream, cudaStreamNonBlocking));
    cudaStream_t s2 = ctx.aux_stream;
    int* nonfinite = dev<int>(ctx.flag, 1);
    double2* Sbuf = dev<double2>(ctx.sk_S, size_t(l) * size_t(m));
    double2* Ebuf = dev<double2>(ctx.sk_E, size_t(l) * size_t(m));
    double qr_s0 = 0.0, qr_s1 = 0.0;
    const double t_sol0 = now_s();
    double t0 = t_sol0;

    // ---- Step 1 (and Step 4's sketch): S = T A^*, E = T' A^*  (src/solver.cpp:80-81, src/lsq.cpp:55-56)
    MNB_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), s1));
    cudaEvent_t eA = ctx.timer_event(), eS = ctx.timer_event(), eE = ctx.timer_event();
    MNB_CUDA(cudaEventRecord(eA, s1));
    // E's Gram block by block while E is sketched in row slabs (c5; the host-A path at c4): after the
    // slab of rows [s0, s0 + rs) lands, G[0:s0+rs, s0:s0+rs] = E[:, :s0+rs]^H E[:, s0:s0+rs] on its own
    // stream, so QR(E) starts from a finished Gram instead of a 16384 x 4096 HERK after the sketch
    double2* GE = nullptr;
    double2* GS = nullptr;  // S's Gram the same way on the host-A path (m > 1024: QR(S) is what remains after the copy)
    bool gram_partial = false;
    cudaEvent_t eG = ctx.timer_event(), eGS = ctx.timer_event();
    auto gram_slab_of = [&](const double2* sketch, DevBuf& store, double2*& Gout, cudaEvent_t done) {
        return [&, sketch, done](int64_t s0, int64_t rs) {
            if (s0 == 0 && rs == m) {  // one slab: nothing to overlap, the QR takes its own HERK
                gram_partial = true;
                return;
            }
            if (!ctx.gram_stream) MNB_CUDA(cudaStreamCreateWithFlags(&ctx.gram_stream, cudaStreamNonBlocking));
            Gout = dev<double2>(store, size_t(m) * size_t(m));
            cudaEvent_t e = ctx.timer_event();
            MNB_CUDA(cudaEventRecord(e, s1));
            MNB_CUDA(cudaStreamWaitEvent(ctx.gram_stream, e, 0));
            const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
            cublasSetStream(ctx.cublas, ctx.gram_stream);
            const cublasStatus_t st = cublasZgemm(ctx.cublas, CUBLAS_OP_C, CUBLAS_OP_N, int(s0 + rs), int(rs), int(l), &one,
                                                  reinterpret_cast<const cuDoubleComplex*>(sketch), int(l),
                                                  reinterpret_cast<const cuDoubleComplex*>(sketch + s0 * l), int(l), &zero,
                                                  reinterpret_cast<cuDoubleComplex*>(Gout + s0 * m), int(m));
            cublasSetStream(ctx.cublas, ctx.stream);
            cublas_check(st, "zgemm (Gram of a sketch)");
            MNB_CUDA(cudaEventRecord(done, ctx.gram_stream));
        };
    };
    const std::function<void(int64_t, int64_t)> gram_slab = gram_slab_of(Ebuf, ctx.gram_E, GE, eG);
    const std::function<void(int64_t, int64_t)> gram_slab_S = gram_slab_of(Sbuf, ctx.gram_Sk, GS, eGS);
    const bool incr_gram = !ctx.distributed() && !std::getenv("MNB_GRAM_AFTER");
    // (S: only where QR(S) takes the host-steered CholeskyQR that honours a precomputed Gram, m > 1024)
    const bool incr_gram_S = incr_gram && pipelined && m > 1024 && !std::getenv("MNB_GRAM_S_AFTER");
    struct SlabHookGuard {  // the hook captures this frame: never let it outlive the solve
        Context& c;
        ~SlabHookGuard() { c.on_slab = nullptr; }
    } slab_hook_guard{ctx};
    if (pipelined) {
        for (size_t k = 0; k < slabs.size(); ++k) {
            const auto [r0, rows] = slabs[k];
            MNB_CUDA(cudaStreamWaitEvent(s1, ctx.event(200 + k), 0));
            ctx.nonfinite = nonfinite;  // the first H stage checks every entry of A as it streams it
            if (incr_gram_S) ctx.on_slab = gram_slab_S;
            sketch_block(ctx, Td, ctx.A, ctx.dtype == MNB_F64, m, r0, rows, Sbuf, l, r0, rep.sketch_kernel_ms);
            ctx.on_slab = nullptr;
            ctx.nonfinite = nullptr;
            if (incr_gram) ctx.on_slab = gram_slab;
            sketch_block(ctx, Tpd, ctx.A, ctx.dtype == MNB_F64, m, r0, rows, Ebuf, l, r0, rep.sketch_kernel_ms);
            ctx.on_slab = nullptr;
            MNB_CUDA(cudaEventRecord(ctx.event(240 + k), s1));
            if (k == 0) trace("slab 0 sketches issued");
        }
        MNB_CUDA(cudaEventRecord(eS, s1));
        MNB_CUDA(cudaEventRecord(eE, s1));
        ctx.pending_host = false;
        ctx.A_host = nullptr;
    } else {
        if (staged) {
            upload_srft_first(ctx, T, Td);
            ctx.after_first_stage = [&] {
                trace("first H stage of S issued");
                fut_T.get();  // the rest of T (rethrows the builder's error)
                if (!ctx.copy_stream) MNB_CUDA(cudaStreamCreateWithFlags(&ctx.copy_stream, cudaStreamNonBlocking));
                upload_srft_rest(ctx, T, Td, ctx.copy_stream, ctx.event(232));
            };
        } else {
            upload_srft(ctx, T, Td);
        }
        ctx.nonfinite = nonfinite;
        trace("upload T issued");
        sketch_matrix(ctx, Td, Sbuf, rep.sketch_kernel_ms, &rep.redistribute_seconds);
        if (ctx.after_first_stage) {  // no local rows to sketch (a rank without a row block)
            auto hook = std::move(ctx.after_first_stage);
            ctx.after_first_stage = nullptr;
            hook();
        }
        ctx.nonfinite = nullptr;
        if (ctx.distributed())  // every rank flagged its own row block
            nccl_check(ncclAllReduce(nonfinite, nonfinite, 1, ncclInt, ncclMax, ctx.comm, s1), "ncclAllReduce");
        MNB_CUDA(cudaEventRecord(eS, s1));
        trace("sketch S issued");
        // E's sketch queues behind S's on s1 (from the same redistributed slab) while s2 factors S
        fut_Tp.get();
        // T' goes up (and its device tables are built) on the copy stream beside S's sketch; queued
        // on s1 the 88 n bytes would land only after S's last kernel, in front of E's first
        // (m <= 1024 -- c3: 32.34 -> 32.1 ms; at c5 the table kernels beside S's sketch and the earlier
        // start of E's sketch against QR(S)'s Gram cost 6 ms, at c4 nothing changes: profiles/r02/ab2;
        // MNB_SIDE_UPLOAD=0 / 1 forces it off / on)
        static const int side_env = std::getenv("MNB_SIDE_UPLOAD") ? std::atoi(std::getenv("MNB_SIDE_UPLOAD")) : -1;
        const bool side_upload = side_env >= 0 ? side_env != 0 : m <= 1024;
        if (side_upload) {
            if (!ctx.copy_stream) MNB_CUDA(cudaStreamCreateWithFlags(&ctx.copy_stream, cudaStreamNonBlocking));
            OnStream on(ctx, ctx.copy_stream);
            upload_srft(ctx, Tp, Tpd);
            MNB_CUDA(cudaEventRecord(ctx.event(233), ctx.copy_stream));
            MNB_CUDA(cudaStreamWaitEvent(s1, ctx.event(233), 0));
        } else {
            upload_srft(ctx, Tp, Tpd);
        }
        if (incr_gram) ctx.on_slab = gram_slab;
        sketch_matrix(ctx, Tpd, Ebuf, rep.sketch_kernel_ms, &rep.redistribute_seconds);
        ctx.on_slab = nullptr;
        MNB_CUDA(cudaEventRecord(eE, s1));
    }
    if (gram_partial) GE = GS = nullptr;  // a single slab after all
    trace("sketch E issued");

    // ---- QR(E) (Step 4's preconditioner, src/lsq.cpp:58-64) on a helper host thread with its own
    // stream, handles and workspaces, beside QR(S) and Steps 2-3 below (whose host round trips would
    // otherwise hold it back until c is ready).  Not at m > 2048 (c5: the S chain finishes during
    // E's sketch anyway, and the duplicated QR workspaces would eat into the sketch's slab budget).
    SketchQr eq;
    cudaEvent_t eQ = ctx.timer_event();
    std::atomic<int> s_verdict{0};  // (declared before the join guard: the helper thread reads it)
    std::future<void> fut_eq;
    struct JoinEq {
        std::future<void>& f;
        ~JoinEq() { if (f.valid()) f.wait(); }
    } join_eq{fut_eq};
    const bool qr_thread = m <= 2048 && !std::getenv("MNB_QR_SERIAL");
    Context* qctx = qr_thread ? &ctx.helper() : nullptr;
    auto qr_E = [&](Context& q) {
        if (GE) MNB_CUDA(cudaStreamWaitEvent(q.stream, eG, 0));
        struct PreGram {
            Context& q;
            PreGram(Context& c, const double2* g) : q(c) { q.pre_gram = g; }
            ~PreGram() { q.pre_gram = nullptr; }
        } pre_gram{q, GE};
        eq = qr_of_sketch(q, Ebuf, l, q.tau_E, q.R_E, &qr_s1, /*precond=*/true, false, double(n));
        if (int64_t bad = eq.deficient >= 0 ? eq.deficient : deficient_count(q, eq.R, eq.ldR, m, n); bad > 0)
            throw Error(MNB_ERR_RANK_DEFICIENCY,
                        "solve_least_squares: sketch QR found " + std::to_string(bad) +
                            " numerically dependent columns",
                        bad);
        MNB_CUDA(cudaEventRecord(eQ, q.stream));
    };
    // what QR(S)'s first Cholesky found (0 not known yet, 1 usable, 2 the sketch needs the shifted
    // chain): E = T' A^* has the same conditioning, so QR(E) skips its own doomed first attempt when
    // the answer is there before E's sketch is (c3: ~2.7 ms of the E chain).  Only worth a wait at
    // m >= 512 -- below, the attempt costs less than the launch latency the wait exposes.
    if (qr_thread) {
        qctx->timers.clear();
        qctx->timer_next = 0;
        qctx->qr_shifted = false;
        MNB_CUDA(cudaStreamWaitEvent(qctx->stream, eE, 0));
        const int device = ctx.device;
        const bool wait_verdict = m >= 512 && !std::getenv("MNB_NO_VERDICT");
        fut_eq = host_async([&, device, wait_verdict] {
            MNB_CUDA(cudaSetDevice(device));
            if (wait_verdict) {
                while (s_verdict.load(std::memory_order_acquire) == 0 && cudaEventQuery(eE) == cudaErrorNotReady)
                    std::this_thread::sleep_for(std::chrono::microseconds(20));
                if (s_verdict.load(std::memory_order_acquire) == 2) qctx->qr_shifted = true;
            }
            qr_E(*qctx);
        });
    }

    // ---- Step 1 QR and Steps 2-3 on s2
    SketchQr sq;
    double2* c_vec = dev<double2>(ctx.vec_n[2], size_t(n));
    double2* z = dev<double2>(ctx.rhs, size_t(l));
    cudaEvent_t eC = ctx.timer_event();
    {
        OnStream on(ctx, s2);
        MNB_CUDA(cudaStreamWaitEvent(s2, eS, 0));
        // QR(S), Step 2 and Step 3 queued back to back on the hand-written kernels (Gram, Cholesky,
        // R1^{-1}, the corrected-seminormal loop, T^* z): the host reads their verdict once.  When the
        // sketch is too ill-conditioned for one Cholesky pass (pivot failure, diagonal ratio, the
        // corrections stall above the rounding level) the host-steered chain below takes over,
        // starting at shifted CholeskyQR3 -- exactly where it would have ended up.
        bool fast_done = false;
        // (m <= 1024: beyond that this chain runs beside E's sketch for tens of milliseconds, and the
        // many-barrier refinement kernel, spinning while only part of its grid is resident, held
        // SMs the sketch's persistent kernels were waiting for: E's sketch +2.3 ms at c4, +13 ms at
        // c5, profiles/r02/s4e.  There the host-steered chain below -- the same Cholesky kernel, cuBLAS
        // GEMV / TRSV calls for the corrections -- stays; MNB_FASTQR_ALL=1 lifts the limit.)
        static const bool fast_all = std::getenv("MNB_FASTQR_ALL") != nullptr;
        if (ctx.fastqr && !ctx.qr_lib && ctx.cholqr && ctx.csne && !ctx.qr_shifted && (m <= 1024 || fast_all)) {
            cudaEvent_t q1 = ctx.timer_event(), q2 = ctx.timer_event();
            MNB_CUDA(cudaEventRecord(q1, ctx.stream));
            DevTrace dt(ctx, "QR(S) + steps 2-3");
            double2* G0 = dev<double2>(ctx.R_S, size_t(m) * size_t(m));
            // (m >= 512: one more host read, after the Cholesky alone, spares an ill-conditioned
            // sketch -- c3 -- the inverse, the corrections and T^* z of a factor it discards: 2 ms)
            static const bool early_on = !(std::getenv("MNB_EARLY_VERDICT") && std::atoi(std::getenv("MNB_EARLY_VERDICT")) == 0);
            const bool usable = launch_fast_step2(ctx, Sbuf, l, m, b_host, z, &dt, G0, early_on && m >= 512);
            MNB_CUDA(cudaEventRecord(q2, ctx.stream));
            if (usable) {
                srft_adjoint_vec(ctx, Td, z, c_vec);
                dt.mark("T^* z");
                MNB_CUDA(cudaEventRecord(eC, ctx.stream));
            }
            int* flag_h = static_cast<int*>(ctx.pin_small.ensure(sizeof(CgState) + 64)) + (sizeof(CgState) + 32) / 4;
            MNB_CUDA(cudaMemcpyAsync(flag_h, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
            const QrStatus& h = read_qr_status(ctx);
            trace("QR(S) + steps 2-3 (one read)");
            dt.dump();
            if (*flag_h) throw Error(MNB_ERR_DIMENSION, "matrix and right-hand side entries must be finite");
            float qms = 0.f;
            MNB_CUDA(cudaEventElapsedTime(&qms, q1, q2));
            qr_s0 += qms * 1e-3;
            const double ratio = h.chol.dmin > 0.0 ? h.chol.dmax / h.chol.dmin : 1e300;
            if (h.chol.info == 0 && !(kEps * ratio * ratio > 1e-3)) {
                if (h.chol.deficient > 0)
                    throw Error(MNB_ERR_RANK_DEFICIENCY,
                                "sketch S = T A* lost rank (" + std::to_string(h.chol.deficient) +
                                    " dependent columns); the problem matrix is rank deficient",
                                h.chol.deficient);
                fast_done = h.ref.accepted != 0;
            }
            if (std::getenv("MNB_TRACE"))
                std::fprintf(stderr, "[mnb] fast QR(S): info %d, diag ratio %.2e, csne %d corrections, ||b - S^H z|| %.3e (thr %.3e) -> %s\n",
                             h.chol.info, ratio, h.ref.iterations, h.ref.best, h.ref.thr * h.ref.nz_best,
                             fast_done ? "accepted" : "fallback");
            int fast_path = 4;
            s_verdict.store(fast_done ? 1 : 2, std::memory_order_release);
            if (!fast_done && !std::getenv("MNB_NO_CHAIN")) {
                // u cond(S)^2 is not small (c3): the shifted two-pass chain gives X = (R2 R1)^{-1} with
                // S X orthonormal to ~1e-8, and the same seminormal loop converges on it in one or two
                // corrections to the Householder-level floor (path 6)
                DevTrace dt2(ctx, "shifted chain (S) + steps 2-3");
                MNB_CUDA(cudaEventRecord(q1, ctx.stream));
                const ShiftedChain ch = launch_shifted_chain(ctx, Sbuf, l, m, G0, double(l), &dt2);
                QrStatus* qs = qr_status_dev(ctx);
                RefineArgs ra;
                ra.mode = REFINE_CSNE;
                ra.S = Sbuf;
                ra.l = l;
                ra.m = m;
                ra.X = ch.X;
                ra.chol = &qs->chol1;
                ra.b = ctx.vec_m[6].as<double2>();  // b, uploaded by the first attempt
                ra.z = z;
                refine_scratch(ctx, ra);
                ra.st = &qs->ref;
                launch_sketch_refine(ra, ctx.num_sms, ctx.stream);
                dt2.mark("csne");
                ctx.launches += 1;
                MNB_CUDA(cudaEventRecord(q2, ctx.stream));
                srft_adjoint_vec(ctx, Td, z, c_vec);
                dt2.mark("T^* z");
                MNB_CUDA(cudaEventRecord(eC, ctx.stream));
                const QrStatus h2 = read_qr_status(ctx);
                trace("shifted chain (S) + steps 2-3 (one read)");
                dt2.dump();
                MNB_CUDA(cudaEventElapsedTime(&qms, q1, q2));
                qr_s0 += qms * 1e-3;
                if (shifted_chain_ok(h2)) {
                    if (h2.chol1.deficient > 0)
                        throw Error(MNB_ERR_RANK_DEFICIENCY,
                                    "sketch S = T A* lost rank (" + std::to_string(h2.chol1.deficient) +
                                        " dependent columns); the problem matrix is rank deficient",
                                    h2.chol1.deficient);
                    fast_done = h2.ref.accepted != 0;
                    fast_path = 6;
                }
                if (std::getenv("MNB_TRACE"))
                    std::fprintf(stderr, "[mnb] shifted chain (S): info %d/%d, diag ratios %.2e/%.2e, csne %d corrections, ||b - S^H z|| %.3e (thr %.3e) -> %s\n",
                                 h2.chol1.info, h2.chol.info, h2.chol1.dmax / h2.chol1.dmin, h2.chol.dmax / h2.chol.dmin,
                                 h2.ref.iterations, h2.ref.best, h2.ref.thr * h2.ref.nz_best,
                                 fast_done ? "accepted" : "fallback");
            }
            if (fast_done) {
                sq = SketchQr{Sbuf, nullptr, ctx.gram.as<double2>(), m, false};
                sq.path = fast_path;
                rep.step_seconds[0] = now_s() - t0;
            } else {
                ctx.qr_shifted = true;
            }
        }
        if (!fast_done) {
        {
            struct PreGramS {  // S's Gram built slab by slab during the copy (host-A path)
                Context& c;
                PreGramS(Context& ctx_, const double2* g) : c(ctx_) { c.pre_gram = g; }
                ~PreGramS() { c.pre_gram = nullptr; }
            } pre_gram_S{ctx, GS};
            if (GS) MNB_CUDA(cudaStreamWaitEvent(ctx.stream, eGS, 0));
            sq = qr_of_sketch(ctx, Sbuf, l, ctx.tau_S, ctx.R_S, &qr_s0, false, /*seminormal=*/true);
        }
        if (s_verdict.load() == 0) s_verdict.store(ctx.qr_shifted ? 2 : 1, std::memory_order_release);
    trace("QR(S)");
        int flag = 0;  // ProblemInstance::validate's finiteness of A, flagged by the first H stage
        MNB_CUDA(cudaMemcpyAsync(&flag, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
        sync(ctx);
        if (flag) throw Error(MNB_ERR_DIMENSION, "matrix and right-hand side entries must be finite");
        rep.step_seconds[0] = now_s() - t0;

        // ---- Step 2: z = Q [R^{-H} b; 0]  (src/solver.cpp:85-97)
        t0 = now_s();
        if (int64_t bad = deficient_count(ctx, sq.R, sq.ldR, m, l); bad > 0)
            throw Error(MNB_ERR_RANK_DEFICIENCY,
                        "sketch S = T A* lost rank (" + std::to_string(bad) +
                            " dependent columns); the problem matrix is rank deficient",
                        bad);
        if (sq.path == 4 && !step2_z_csne(ctx, sq, Sbuf, b_host, l, m, z)) {
            ctx.qr_shifted = true;  // u cond(S)^2 is not small: CholeskyQR2 would not be accurate either
            sq = qr_of_sketch(ctx, Sbuf, l, ctx.tau_S, ctx.R_S, &qr_s0);  // the full factorization
            if (int64_t bad = deficient_count(ctx, sq.R, sq.ldR, m, l); bad > 0)
                throw Error(MNB_ERR_RANK_DEFICIENCY,
                            "sketch S = T A* lost rank (" + std::to_string(bad) +
                                " dependent columns); the problem matrix is rank deficient",
                            bad);
        }
        if (sq.path != 4) step2_z(ctx, sq, b_host, l, m, z);
        sync(ctx);
        rep.step_seconds[1] = now_s() - t0;

        // ---- Step 3: c = T^* z  (src/solver.cpp:100-102)
        t0 = now_s();
        srft_adjoint_vec(ctx, Td, z, c_vec);
        MNB_CUDA(cudaEventRecord(eC, ctx.stream));
        sync(ctx);
        rep.step_seconds[2] = now_s() - t0;
        }
    }
    trace("steps 2-3");
    const double2* c_loc = c_vec + ctx.col_begin;

    // ---- Step 4: y = argmin ||A^* y - c||  (src/solver.cpp:104-114, src/lsq.cpp:43-113)
    t0 = now_s();
    rep.param_seconds = t_param_T + t_param_Tp;
    double2* y = dev<double2>(ctx.vec_m[5], size_t(m));
    double2* ax = dev<double2>(ctx.vec_m[7], size_t(m));
    double2* xacc = ctx.n_local ? x_dev : nullptr;
    // the INIT pass (r = c, s = A c) needs only c: on s1 while s2 factors E
    MNB_CUDA(cudaStreamWaitEvent(s1, eC, 0));
    // (A c = S^H z needs the sketch intact: not after the Householder fallback, which overwrote it)
    if (sq.path != 2 && !std::getenv("MNB_INIT_PASS")) launch_cg_init_from_sketch(ctx, Sbuf, l, z, c_loc, xacc);
    else launch_cg_init_pass(ctx, c_loc, xacc);
    trace("INIT issued");
    if (qr_thread) {
        fut_eq.get();  // rethrows the helper's errors
        ctx.launches += qctx->launches;
        qctx->launches = 0;
    } else {
        OnStream on(ctx, s2);
        MNB_CUDA(cudaStreamWaitEvent(s2, eE, 0));
        qr_E(ctx);
    }
    trace("QR(E)");
    MNB_CUDA(cudaStreamWaitEvent(s1, eQ, 0));
    LsqResult ls = run_cg(ctx, c_loc, eq.R, eq.ldR, rep.lsq_tau, cfg.lsq_max_iterations, double(Tp.max_mult), y, false,
                          xacc, ax, /*init_done=*/true, eq.rinv_ready, qr_thread ? qctx->Rinv.as<double2>() : nullptr);
    trace("CG");
    {
        float ms = 0.f;
        MNB_CUDA(cudaEventElapsedTime(&ms, eA, eS));
        rep.sketch_seconds[0] = ms * 1e-3;
        MNB_CUDA(cudaEventElapsedTime(&ms, eS, eE));
        rep.sketch_seconds[1] = ms * 1e-3;  // pipelined: 0 (both sketches are interleaved in [0])
    }
    rep.qr_seconds[0] = qr_s0;
    rep.qr_seconds[1] = qr_s1;
    rep.qr_path = sq.path | (eq.path << 4);
    rep.lsq_iterations = ls.iterations;
    rep.lsq_converged = ls.converged ? 1 : 0;
    rep.lsq_achieved_excess = ls.achieved_excess;
    rep.pcg_seconds = ls.pcg_seconds;
    rep.pcg_pass_ms_sum = ls.pass_ms;
    rep.pcg_pass_launches = ls.pass_launches;
    rep.step_seconds[3] = now_s() - t0;

    // ---- Step 5: x = A^* y, residual ||A x - b|| (src/solver.cpp:118-125).  x and A x were
    // accumulated inside the CG passes (x = sum_k alpha_k t_k, A x = sum_k alpha_k s_k): no extra pass.
    t0 = now_s();
    std::vector<double> axh(size_t(2 * m));
    MNB_CUDA(cudaMemcpyAsync(axh.data(), ax, size_t(m) * 16, cudaMemcpyDeviceToHost, ctx.stream));
    if (c_dev && ctx.n_local)
        MNB_CUDA(cudaMemcpyAsync(c_dev, c_loc, size_t(ctx.n_local) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
    sync(ctx);
    rep.step_seconds[4] = now_s() - t0;
    double res2 = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        const double dr = axh[size_t(2 * i)] - reinterpret_cast<const double*>(b_host)[2 * i];
        const double di = axh[size_t(2 * i + 1)] - reinterpret_cast<const double*>(b_host)[2 * i + 1];
        res2 += dr * dr + di * di;
    }
    rep.residual_norm = std::sqrt(res2);
    const double xnorm = std::sqrt(ls.xx);
    rep.c_norm_ratio = xnorm > 0.0 ? std::sqrt(ls.rr0) * std::sqrt(double(l) / (cfg.alpha * double(n))) / xnorm : 0.0;
    ctx.resolve_timers();
    trace("resolve");
    if (!pipelined && std::getenv("MNB_TRACE")) {  // device timeline from the first sketch kernel
        float a = 0.f, b = 0.f, c = 0.f, d = 0.f;
        MNB_CUDA(cudaEventElapsedTime(&a, eA, eS));
        MNB_CUDA(cudaEventElapsedTime(&b, eA, eE));
        MNB_CUDA(cudaEventElapsedTime(&c, eA, eC));
        MNB_CUDA(cudaEventElapsedTime(&d, eA, eQ));
        std::fprintf(stderr, "[mnb] device: sketch S done %.1f ms, sketch E done %.1f, c ready %.1f, R' ready %.1f ms\n",
                     a, b, c, d);
        if (staged)
            std::fprintf(stderr, "[mnb] staged draw of T: first half ready %.2f ms, whole T %.2f ms after the solve began to draw\n",
                         1e3 * t_first_T, 1e3 * t_param_T);
    }
    if (pipelined && std::getenv("MNB_TRACE")) {  // device timeline of the host-A path
        float ms_h2d = 0.f, ms_s = 0.f, ms_c = 0.f, ms_q = 0.f;
        cudaEvent_t e0 = ctx.event(199);
        MNB_CUDA(cudaEventElapsedTime(&ms_h2d, e0, ctx.event(200 + slabs.size() - 1)));
        MNB_CUDA(cudaEventElapsedTime(&ms_s, e0, eE));
        MNB_CUDA(cudaEventElapsedTime(&ms_c, e0, eC));
        MNB_CUDA(cudaEventElapsedTime(&ms_q, e0, eQ));
        std::fprintf(stderr, "[mnb] device: H2D done %.1f ms, sketches done %.1f, c ready %.1f, R' ready %.1f ms\n",
                     ms_h2d, ms_s, ms_c, ms_q);
        {
            float a = 0.f, b = 0.f;
            MNB_CUDA(cudaEventElapsedTime(&a, e0, ctx.event(230)));
            MNB_CUDA(cudaEventElapsedTime(&b, e0, ctx.event(231)));
            std::fprintf(stderr, "[mnb]   T uploaded %.1f ms, T' uploaded %.1f ms\n", a, b);
        }
        for (size_t k = 0; k < slabs.size(); ++k) {
            float a = 0.f, b = 0.f;
            MNB_CUDA(cudaEventElapsedTime(&a, e0, ctx.event(200 + k)));
            MNB_CUDA(cudaEventElapsedTime(&b, e0, ctx.event(240 + k)));
            std::fprintf(stderr, "[mnb]   slab %zu: landed %.1f ms, sketched %.1f ms\n", k, a, b);
        }
    }
    rep.kernel_launches = ctx.launches - launches0;
    rep.total_seconds = now_s() - t_start;
}

// ------------------------------------------------- apply_adjoint_matrix ----
// x = A^H y (this rank's columns) and A x (over all ranks) in one fused pass: Step 5 of the
// solve (src/solver.cpp:118-125) as a standalone product.
void apply_adjoint_matrix(Context& ctx, const void* y, bool y_on_device, double2* x_dev, double2* ax_host) {
    validate_matrix_set(ctx);
    const int64_t m = ctx.m, nl = ctx.n_local;
    double2* yd = dev<double2>(ctx.vec_m[0], size_t(m));
    MNB_CUDA(cudaMemcpyAsync(yd, y, size_t(m) * 16, y_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                             ctx.stream));
    PassBuffers pb = pass_buffers(ctx);
    double2* t = dev<double2>(ctx.vec_n[1], size_t(std::max<int64_t>(nl, 1)));
    fused_pass(ctx, pb, PCG_APPLY, yd, nullptr, nl ? x_dev : t, nullptr, nullptr);
    if (ax_host) MNB_CUDA(cudaMemcpyAsync(ax_host, pb.red, size_t(m) * 16, cudaMemcpyDeviceToHost, ctx.stream));
    sync(ctx);
}

// ------------------------------------------------------ solve_classical ----
// solve_classical (src/solver.cpp:130-146): the deterministic O(m^2 n) baseline.  See
// include/minnorm_b200.h for the two paths.  Path 0 is the Gram-matrix form of the same
// minimal-norm solution, x = A^H (A A^H)^{-1} b, made as accurate as the QR form by corrections
// (each one fused pass: t = A^H z and A t in one read of A); path 1 is the reference's
// Householder QR of A^H without the column pivoting (a full-rank A needs none for x).
void solve_classical(Context& ctx, const double2* b_host, double2* x_dev, mnb_classical_report& rep) {
    const double t_start = now_s();
    validate_matrix_set(ctx);
    rep = mnb_classical_report{};
    const int64_t m = ctx.m, n = ctx.n_global;
    if (m < 1 || m >= n)
        throw Error(MNB_ERR_DIMENSION, "problem must be underdetermined: 1 <= m < n, got m=" + std::to_string(m) +
                                           ", n=" + std::to_string(n));
    bool b_zero = true, b_finite = true;
    for (int64_t i = 0; i < 2 * m; ++i) {
        const double v = reinterpret_cast<const double*>(b_host)[i];
        b_finite = b_finite && std::isfinite(v);
        b_zero = b_zero && v == 0.0;
    }
    if (!b_finite) throw Error(MNB_ERR_DIMENSION, "matrix and right-hand side entries must be finite");
    ctx.make_resident();
    const int64_t nl = ctx.n_local;
    if (b_zero) {  // src/solver.cpp:134
        if (nl) MNB_CUDA(cudaMemsetAsync(x_dev, 0, size_t(nl) * 16, ctx.stream));
        sync(ctx);
        rep.seconds = now_s() - t_start;
        return;
    }
    const auto* Ac = reinterpret_cast<const cuDoubleComplex*>(ctx.A);
    double2* G = dev<double2>(ctx.gram, size_t(m) * size_t(m));
    int* info = dev<int>(ctx.qr_info, 2);
    // ---- path 0: G = A A^H = R1^H R1
    bool ok = true;
    {
        const double one = 1.0, zero = 0.0;
        if (nl && ctx.dtype == MNB_F64) {  // real A: G = A A^T by DSYRK, widened to the complex G
            double* Gr = dev<double>(ctx.qwork, size_t(m) * size_t(m));
            cublas_check(cublasDsyrk(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, int(m), int(nl), &one,
                                     static_cast<const double*>(ctx.A), int(m), &zero, Gr, int(m)),
                         "dsyrk");
            launch_real_to_complex(Gr, G, m * m, ctx.stream);
            ctx.launches += 1;
        } else if (nl) {
            cublas_check(cublasZherk(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, int(m), int(nl), &one, Ac, int(m),
                                     &zero, reinterpret_cast<cuDoubleComplex*>(G), int(m)),
                         "zherk");
        } else {
            MNB_CUDA(cudaMemsetAsync(G, 0, size_t(m) * size_t(m) * 16, ctx.stream));
        }
        allreduce_sum(ctx, reinterpret_cast<double*>(G), size_t(2 * m * m));
        size_t dws = 0, hws = 0;
        cusolver_check(cusolverDnXpotrf_bufferSize(ctx.cusolver, ctx.cusolver_params, CUBLAS_FILL_MODE_UPPER, m,
                                                   CUDA_C_64F, G, m, CUDA_C_64F, &dws, &hws),
                       "potrf_bufferSize");
        void* work = ctx.qr_work.ensure(std::max<size_t>(dws, 16));
        if (ctx.host_work.size() < hws + 16) ctx.host_work.resize(hws + 16);
        cusolver_check(cusolverDnXpotrf(ctx.cusolver, ctx.cusolver_params, CUBLAS_FILL_MODE_UPPER, m, CUDA_C_64F, G, m,
                                        CUDA_C_64F, work, dws, ctx.host_work.data(), hws, info),
                       "potrf");
        int info_h = 0;
        std::vector<double> diag(size_t(2 * m));
        MNB_CUDA(cudaMemcpyAsync(&info_h, info, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
        MNB_CUDA(cudaMemcpy2DAsync(diag.data(), 16, G, size_t(m + 1) * 16, 16, size_t(m), cudaMemcpyDeviceToHost,
                                   ctx.stream));
        sync(ctx);
        double dmax = 0.0, dmin = 1e300;
        for (int64_t j = 0; j < m; ++j) {
            const double a = std::hypot(diag[size_t(2 * j)], diag[size_t(2 * j + 1)]);
            dmax = std::max(dmax, a);
            dmin = std::min(dmin, a);
        }
        ok = info_h == 0 && dmin > 0.0 && dmax / dmin < 1e7;
    }
    if (ok) {
        launch_zero_lower(G, m, ctx.stream);  // potrf leaves the strict lower triangle unreferenced
        ctx.launches += 1;
        double fro = 0.0;  // ||R1||_F = sqrt(trace G) = ||A||_F
        cublas_check(cublasDznrm2(ctx.cublas, int(m * m), reinterpret_cast<const cuDoubleComplex*>(G), 1, &fro),
                     "dznrm2");
        const double thr = 2.0 * std::sqrt(double(n)) * kEps * fro;  // rounding level of ||A x|| / ||x||
        PassBuffers pb = pass_buffers(ctx);
        double2* zd = dev<double2>(ctx.vec_m[0], size_t(m));
        double2* dx = dev<double2>(ctx.vec_n[1], size_t(std::max<int64_t>(nl, 1)));
        double* scal = dev<double>(ctx.scratch, 1024);
        std::vector<double2> r(b_host, b_host + m), s(static_cast<size_t>(m)), ax(static_cast<size_t>(m));
        double prev = 0.0;
        ok = false;
        // x is kept explicitly and corrected, x_{k+1} = x_k + A^H G^{-1} (b - A x_k) (Bjorck's corrected
        // seminormal equations): each step one fused pass gives dx = A^H dz and A dx together.
        for (int it = 0; it <= 8; ++it) {
            MNB_CUDA(cudaMemcpyAsync(zd, r.data(), size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
            cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, int(m),
                                     reinterpret_cast<const cuDoubleComplex*>(G), int(m),
                                     reinterpret_cast<cuDoubleComplex*>(zd), 1),
                         "ztrsv");
            cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, int(m),
                                     reinterpret_cast<const cuDoubleComplex*>(G), int(m),
                                     reinterpret_cast<cuDoubleComplex*>(zd), 1),
                         "ztrsv");
            fused_pass(ctx, pb, PCG_APPLY, zd, nullptr, it == 0 ? x_dev : dx, nullptr, nullptr);
            MNB_CUDA(cudaMemcpyAsync(s.data(), pb.red, size_t(m) * 16, cudaMemcpyDeviceToHost, ctx.stream));
            if (it > 0 && nl) {
                const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0);
                cublas_check(cublasZaxpy(ctx.cublas, int(nl), &one, reinterpret_cast<const cuDoubleComplex*>(dx), 1,
                                         reinterpret_cast<cuDoubleComplex*>(x_dev), 1),
                             "zaxpy");
            }
            double xn = 0.0;  // ||x||: this rank's part, summed over ranks
            if (nl) cublas_check(cublasDznrm2(ctx.cublas, int(nl), reinterpret_cast<const cuDoubleComplex*>(x_dev), 1, &xn),
                                 "dznrm2");
            xn *= xn;
            MNB_CUDA(cudaMemcpyAsync(scal, &xn, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
            allreduce_sum(ctx, scal, 1);
            MNB_CUDA(cudaMemcpyAsync(&xn, scal, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
            sync(ctx);
            double rn = 0.0;
            for (int64_t i = 0; i < m; ++i) {
                ax[size_t(i)] = it == 0 ? s[size_t(i)]
                                        : make_double2(ax[size_t(i)].x + s[size_t(i)].x, ax[size_t(i)].y + s[size_t(i)].y);
                r[size_t(i)] = make_double2(b_host[i].x - ax[size_t(i)].x, b_host[i].y - ax[size_t(i)].y);
                rn += r[size_t(i)].x * r[size_t(i)].x + r[size_t(i)].y * r[size_t(i)].y;
            }
            rn = std::sqrt(rn);
            rep.refinements = it;
            rep.residual_norm = rn;
            // keep correcting while the residual still halves (the forward error follows it down,
            // times cond(A)); accept once it stagnates at the rounding level of A x
            const bool at_floor = rn <= thr * std::sqrt(xn);
            if (it > 0 && !(rn < 0.5 * prev)) {
                ok = at_floor;  // stagnated: at the floor (done) or above it (u cond(A)^2 too large)
                break;
            }
            if (it == 8) {
                ok = at_floor;
                break;
            }
            prev = rn;
        }
        rep.path = 0;
    }
    if (!ok) {
        // ---- path 1: Householder QR of A^H (the reference's algorithm, src/solver.cpp:130-146), as a
        // TSQR over the ranks' column shards: A^H = diag(Q_J) [R_1; ...; R_w] = diag(Q_J) Q~ R.
        //   1. each rank: Householder QR of its n_J x m block A_J^H -> reflectors + R_J
        //   2. allgather the R_J (m x m each) and factor the stack (w m x m) -> Q~, R (replicated)
        //   3. rank rule on the singular values of R (rank-revealing, unlike the unpivoted R_jj):
        //      sigma_j < n eps sigma_max counts as dependent, the reference's threshold
        //      (src/solver.cpp:137-140 on its column-pivoted R)
        //   4. x = diag(Q_J) Q~ [R^{-H} b; 0]: v = Q~ [w; 0] (replicated), x_J = Q_J [v_J; 0]
        // One GPU is the w = 1 case (Q~ = I).  Real A is widened to complex per shard.
        const int world = ctx.distributed() ? ctx.world : 1;
        const int64_t kq = std::min<int64_t>(nl, m);  // rows of R_J that the local QR defines
        double2* AH = dev<double2>(ctx.ws_x1, size_t(std::max<int64_t>(nl, 1)) * size_t(m));
        if (nl) {
            if (ctx.dtype == MNB_F64) {
                double2* Aw = dev<double2>(ctx.ws_x2, size_t(m) * size_t(nl));
                launch_real_to_complex(static_cast<const double*>(ctx.A), Aw, m * nl, ctx.stream);
                launch_transpose(Aw, m, nl, m, AH, nl, ctx.stream);
            } else {
                launch_transpose(static_cast<const double2*>(ctx.A), m, nl, m, AH, nl, ctx.stream);
            }
            launch_conj_inplace(AH, nl * m, ctx.stream);
            ctx.launches += 3;
        }
        double2* tau = dev<double2>(ctx.tau_S, size_t(m));
        auto geqrf = [&](double2* M, int64_t rows, int64_t ld, double2* t) {
            size_t dws = 0, hws = 0;
            cusolver_check(cusolverDnXgeqrf_bufferSize(ctx.cusolver, ctx.cusolver_params, rows, m, CUDA_C_64F, M, ld,
                                                       CUDA_C_64F, t, CUDA_C_64F, &dws, &hws),
                           "geqrf_bufferSize");
            void* work = ctx.qr_work.ensure(std::max<size_t>(dws, 16));
            if (ctx.host_work.size() < hws + 16) ctx.host_work.resize(hws + 16);
            cusolver_check(cusolverDnXgeqrf(ctx.cusolver, ctx.cusolver_params, rows, m, CUDA_C_64F, M, ld, CUDA_C_64F,
                                            t, CUDA_C_64F, work, dws, ctx.host_work.data(), hws, info),
                           "geqrf");
        };
        auto unmqr = [&](const double2* M, int64_t rows, int64_t ld, const double2* t, int64_t k, double2* v) {
            int lwork = 0;
            cusolver_check(cusolverDnZunmqr_bufferSize(ctx.cusolver, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, int(rows), 1, int(k),
                                                       reinterpret_cast<const cuDoubleComplex*>(M), int(ld),
                                                       reinterpret_cast<const cuDoubleComplex*>(t),
                                                       reinterpret_cast<const cuDoubleComplex*>(v), int(rows), &lwork),
                           "unmqr_bufferSize");
            auto* wk = static_cast<cuDoubleComplex*>(ctx.qr_work.ensure(size_t(std::max(lwork, 1)) * 16));
            cusolver_check(cusolverDnZunmqr(ctx.cusolver, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, int(rows), 1, int(k),
                                            reinterpret_cast<const cuDoubleComplex*>(M), int(ld),
                                            reinterpret_cast<const cuDoubleComplex*>(t), reinterpret_cast<cuDoubleComplex*>(v),
                                            int(rows), wk, lwork, info),
                           "unmqr");
        };
        if (nl) geqrf(AH, nl, nl, tau);
        // R_J (m x m, zero below the diagonal and below row kq) into this rank's block of the stack
        double2* stack = dev<double2>(ctx.R2, size_t(world) * size_t(m) * size_t(m));  // [w][m x m] col-major
        double2* Rj = stack + size_t(world > 1 ? ctx.rank : 0) * size_t(m) * size_t(m);
        MNB_CUDA(cudaMemsetAsync(Rj, 0, size_t(m) * size_t(m) * 16, ctx.stream));
        if (kq) MNB_CUDA(cudaMemcpy2DAsync(Rj, size_t(m) * 16, AH, size_t(nl) * 16, size_t(kq) * 16, size_t(m),
                                           cudaMemcpyDeviceToDevice, ctx.stream));
        launch_zero_lower(Rj, m, ctx.stream);
        ctx.launches += 1;
        double2* R = Rj;  // m x m upper, leading dimension ldR
        int64_t ldR = m;
        double2* Sg = nullptr;  // the factored stack (w m x m, leading dimension w m)
        double2* tau2 = nullptr;
        if (world > 1) {
            nccl_check(ncclAllGather(Rj, stack, size_t(2 * m * m), ncclDouble, ctx.comm, ctx.stream), "ncclAllGather");
            // [w][m x m] blocks -> one (w m) x m column-major matrix
            Sg = dev<double2>(ctx.qwork, size_t(world) * size_t(m) * size_t(m));
            for (int h = 0; h < world; ++h)
                MNB_CUDA(cudaMemcpy2DAsync(Sg + size_t(h) * size_t(m), size_t(world) * size_t(m) * 16,
                                           stack + size_t(h) * size_t(m) * size_t(m), size_t(m) * 16, size_t(m) * 16,
                                           size_t(m), cudaMemcpyDeviceToDevice, ctx.stream));
            tau2 = dev<double2>(ctx.tau_E, size_t(m));
            geqrf(Sg, int64_t(world) * m, int64_t(world) * m, tau2);
            R = Sg;
            ldR = int64_t(world) * m;
        }
        // rank rule on the singular values of R
        {
            double2* Rc = dev<double2>(ctx.gram, size_t(m) * size_t(m));
            MNB_CUDA(cudaMemcpy2DAsync(Rc, size_t(m) * 16, R, size_t(ldR) * 16, size_t(m) * 16, size_t(m),
                                       cudaMemcpyDeviceToDevice, ctx.stream));
            launch_zero_lower(Rc, m, ctx.stream);
            ctx.launches += 1;
            double* sv = dev<double>(ctx.scratch, size_t(std::max<int64_t>(m, 512)));
            size_t dws = 0, hws = 0;
            cusolver_check(cusolverDnXgesvd_bufferSize(ctx.cusolver, ctx.cusolver_params, 'N', 'N', m, m, CUDA_C_64F, Rc,
                                                       m, CUDA_R_64F, sv, CUDA_C_64F, nullptr, 1, CUDA_C_64F, nullptr, 1,
                                                       CUDA_C_64F, &dws, &hws),
                           "gesvd_bufferSize");
            void* work = ctx.qr_work.ensure(std::max<size_t>(dws, 16));
            if (ctx.host_work.size() < hws + 16) ctx.host_work.resize(hws + 16);
            cusolver_check(cusolverDnXgesvd(ctx.cusolver, ctx.cusolver_params, 'N', 'N', m, m, CUDA_C_64F, Rc, m,
                                            CUDA_R_64F, sv, CUDA_C_64F, nullptr, 1, CUDA_C_64F, nullptr, 1, CUDA_C_64F,
                                            work, dws, ctx.host_work.data(), hws, info),
                           "gesvd");
            std::vector<double> svh(static_cast<size_t>(m));
            MNB_CUDA(cudaMemcpyAsync(svh.data(), sv, size_t(m) * 8, cudaMemcpyDeviceToHost, ctx.stream));
            sync(ctx);
            const double smax = *std::max_element(svh.begin(), svh.end());
            const double thr_r = double(n) * kEps * smax;
            int64_t bad = 0;
            for (double v : svh)
                if (!(v >= thr_r) || v == 0.0) ++bad;
            if (bad > 0)
                throw Error(MNB_ERR_RANK_DEFICIENCY,
                            "pivoted QR found rank deficiency (" + std::to_string(bad) + " dependent columns)", bad);
        }
        // w = R^{-H} b, v = Q~ [w; 0] (replicated), x_J = Q_J [v_J; 0]
        double2* v = dev<double2>(ctx.vec_m[9], size_t(world) * size_t(m));
        MNB_CUDA(cudaMemsetAsync(v, 0, size_t(world) * size_t(m) * 16, ctx.stream));
        MNB_CUDA(cudaMemcpyAsync(v, b_host, size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
        cublas_check(cublasZtrsv(ctx.cublas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, int(m),
                                 reinterpret_cast<const cuDoubleComplex*>(R), int(ldR),
                                 reinterpret_cast<cuDoubleComplex*>(v), 1),
                     "ztrsv");
        if (world > 1) unmqr(Sg, int64_t(world) * m, int64_t(world) * m, tau2, m, v);
        if (nl) {
            MNB_CUDA(cudaMemsetAsync(x_dev, 0, size_t(nl) * 16, ctx.stream));
            MNB_CUDA(cudaMemcpyAsync(x_dev, v + size_t(world > 1 ? ctx.rank : 0) * size_t(m), size_t(kq) * 16,
                                     cudaMemcpyDeviceToDevice, ctx.stream));
            unmqr(AH, nl, nl, tau, kq, x_dev);
        }
        // ||A x - b|| through the INIT pass (s = A x, summed over the ranks)
        PassBuffers pb = pass_buffers(ctx);
        double2* r1 = dev<double2>(ctx.vec_n[0], size_t(std::max<int64_t>(nl, 1)));
        double2* t1 = dev<double2>(ctx.vec_n[1], size_t(std::max<int64_t>(nl, 1)));
        fused_pass(ctx, pb, PCG_INIT, nullptr, x_dev, t1, r1, nullptr, nullptr);
        std::vector<double2> s(static_cast<size_t>(m));
        MNB_CUDA(cudaMemcpyAsync(s.data(), pb.red, size_t(m) * 16, cudaMemcpyDeviceToHost, ctx.stream));
        sync(ctx);
        double rn = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            const double dr = b_host[i].x - s[size_t(i)].x, di = b_host[i].y - s[size_t(i)].y;
            rn += dr * dr + di * di;
        }
        rep.path = 1;
        rep.residual_norm = std::sqrt(rn);
    }
    sync(ctx);
    rep.seconds = now_s() - t_start;
}

// ------------------------------------------------ solve_least_squares -----
void solve_least_squares(Context& ctx, const double2* c_dev, const mnb_lsq_config& cfg, double2* y_host,
                         double* residual_norms, mnb_lsq_solution& sol) {
    validate_matrix_set(ctx);
    ctx.timers.clear();
    ctx.timer_next = 0;
    ctx.qr_shifted = false;
    const int64_t m = ctx.m, n = ctx.n_global;  // B = A^H is n x m
    // src/lsq.cpp:45-53
    if (m < 1 || n <= m) throw Error(MNB_ERR_INVALID_ARGUMENT, "solve_least_squares: B must be tall (n > m >= 1)");
    if (cfg.sketch_size <= m || cfg.sketch_size > n)
        throw Error(MNB_ERR_INVALID_ARGUMENT, "solve_least_squares: sketch size must lie in (m, n]");
    if (!(cfg.tau > 0.0)) throw Error(MNB_ERR_INVALID_ARGUMENT, "solve_least_squares: tau must be positive");
    if (cfg.max_iterations < 1)
        throw Error(MNB_ERR_INVALID_ARGUMENT, "solve_least_squares: max_iterations must be at least 1");
    SrftHost Tp;
    build_srft_host(Tp, cfg.sketch_size, n, cfg.stream_seed, cfg.sampling,
                    [&](size_t bytes) { return pinned_alloc(ctx.pin_params[1], bytes); }, [](unsigned char*) {}, 0);
    SrftDev& Tpd = ctx.op_dev[1];
    upload_srft(ctx, Tp, Tpd);
    SketchQr eq = sketch_and_qr(ctx, Tpd, ctx.sk_E, ctx.tau_E, ctx.R_E, nullptr, nullptr, nullptr, nullptr, true);
    if (int64_t bad = deficient_count(ctx, eq.R, eq.ldR, m, n); bad > 0)
        throw Error(MNB_ERR_RANK_DEFICIENCY,
                    "solve_least_squares: sketch QR found " + std::to_string(bad) + " numerically dependent columns",
                    bad);
    double2* y = dev<double2>(ctx.vec_m[5], size_t(m));
    LsqResult ls = run_cg(ctx, c_dev, eq.R, eq.ldR, cfg.tau, cfg.max_iterations, double(Tp.max_mult), y,
                          residual_norms != nullptr, nullptr, nullptr, false, eq.rinv_ready);
    MNB_CUDA(cudaMemcpyAsync(y_host, y, size_t(m) * 16, cudaMemcpyDeviceToHost, ctx.stream));
    sync(ctx);
    sol.achieved_excess = ls.achieved_excess;
    sol.iterations = ls.iterations;
    sol.converged = ls.converged ? 1 : 0;
    if (residual_norms)
        for (size_t i = 0; i < ls.residual_norms.size(); ++i) residual_norms[i] = ls.residual_norms[i];
}

// ----------------------------------------------------------- benchmark ----
double bench_pcg_pass(Context& ctx, int reps) {
    validate_matrix_set(ctx);
    const int64_t m = ctx.m;
    PassBuffers pb = pass_buffers(ctx);
    double2* w = dev<double2>(ctx.vec_m[0], size_t(m));
    std::vector<double> wh(size_t(2 * m));
    for (int64_t i = 0; i < 2 * m; ++i) wh[size_t(i)] = 1.0 / double(1 + i % 7);
    MNB_CUDA(cudaMemcpyAsync(w, wh.data(), size_t(m) * 16, cudaMemcpyHostToDevice, ctx.stream));
    double2* t = dev<double2>(ctx.vec_n[1], size_t(std::max<int64_t>(ctx.n_local, 1)));
    fused_pass(ctx, pb, PCG_APPLY, w, nullptr, t, nullptr, nullptr);  // warm-up
    cudaEvent_t e0 = ctx.event(40), e1 = ctx.event(41);
    MNB_CUDA(cudaEventRecord(e0, ctx.stream));
    for (int i = 0; i < reps; ++i) {
        PcgPassArgs a;
        a.A = ctx.A;
        a.is_real = ctx.dtype == MNB_F64;
        a.m = m;
        a.n = ctx.n_local;
        a.w = w;
        a.tout = t;
        a.part_s = pb.part_s;
        a.part_scal = pb.part_scal;
        a.mode = PCG_APPLY;
        launch_pcg_pass(a, pb.plan, ctx.stream);
        ctx.launches += 1;
    }
    MNB_CUDA(cudaEventRecord(e1, ctx.stream));
    MNB_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    MNB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    return double(ms) / reps;
}

}  // namespace mnb
