// extern "C" boundary (include/minnorm_b200.h): status codes in, exceptions out.
#include <cstdlib>
#include <cstring>
#include <string>

#include "context.cuh"
#include "mm_io.hpp"

struct mnb_context {
    mnb::Context ctx;
};
struct mnb_srft {
    mnb::SrftHost host;
};

namespace {

thread_local std::string g_error;
thread_local int64_t g_deficient = 0;
thread_local int64_t g_parse_line = 0, g_parse_column = 0;

template <class F>
int guard(F&& f) {
    try {
        f();
        return MNB_OK;
    } catch (const mnb::ParseFail& e) {
        g_error = e.what();
        g_parse_line = e.line;
        g_parse_column = e.column;
        return e.code;
    } catch (const mnb::Error& e) {
        g_error = e.what();
        g_deficient = e.deficient;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return MNB_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_error = e.what();
        return MNB_ERR_INTERNAL;
    } catch (...) {
        g_error = "unknown error";
        return MNB_ERR_INTERNAL;
    }
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw mnb::Error(MNB_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

void init_context(mnb::Context& c, int device) {
    int count = 0;
    MNB_CUDA(cudaGetDeviceCount(&count));
    mnb::require(device >= 0 && device < count, MNB_ERR_INVALID_ARGUMENT, "invalid CUDA device index");
    c.device = device;
    MNB_CUDA(cudaSetDevice(device));
    MNB_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
    MNB_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    c.own_stream = true;
    if (const char* q = std::getenv("MNB_QR")) c.cholqr = std::string(q) != "householder";
    if (const char* q = std::getenv("MNB_CSNE")) c.csne = std::string(q) != "0";
    if (const char* q = std::getenv("MNB_P2FA")) c.p2fa = std::string(q) != "0";
    if (const char* q = std::getenv("MNB_PRECOND_2NORM")) c.two_norm_check = std::string(q) != "0";
    if (const char* q = std::getenv("MNB_FASTQR")) c.fastqr = std::string(q) != "0";
    if (const char* q = std::getenv("MNB_QR_LIB")) c.qr_lib = std::string(q) == "1";
    if (cublasCreate(&c.cublas) != CUBLAS_STATUS_SUCCESS) throw mnb::Error(MNB_ERR_CUDA, "cublasCreate failed");
    cublasSetStream(c.cublas, c.stream);
    if (cusolverDnCreate(&c.cusolver) != CUSOLVER_STATUS_SUCCESS) throw mnb::Error(MNB_ERR_CUDA, "cusolverDnCreate failed");
    cusolverDnSetStream(c.cusolver, c.stream);
    if (cusolverDnCreateParams(&c.cusolver_params) != CUSOLVER_STATUS_SUCCESS)
        throw mnb::Error(MNB_ERR_CUDA, "cusolverDnCreateParams failed");
}

}  // namespace

namespace mnb {
std::unique_ptr<Context> make_helper_context(const Context& parent) {
    auto h = std::make_unique<Context>();
    init_context(*h, parent.device);
    h->cholqr = parent.cholqr;
    h->csne = parent.csne;
    h->p2fa = parent.p2fa;
    h->two_norm_check = parent.two_norm_check;
    h->fastqr = parent.fastqr;
    h->qr_lib = parent.qr_lib;
    return h;
}
}  // namespace mnb

namespace {

void copy_out(void* dst, const void* src, size_t bytes, int location, cudaStream_t stream) {
    MNB_CUDA(cudaMemcpyAsync(dst, src, bytes, location == MNB_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             stream));
}

}  // namespace

extern "C" {

const char* mnb_last_error(void) { return g_error.c_str(); }
int64_t mnb_last_deficient_columns(void) { return g_deficient; }
const char* mnb_version(void) { return "minnorm_b200 0.1 (sm_100a)"; }

int mnb_shard_columns(int64_t n, int world_size, int rank, int64_t* col_begin, int64_t* col_count) {
    return guard([&] {
        mnb::require(world_size >= 1 && rank >= 0 && rank < world_size && n >= 0, MNB_ERR_INVALID_ARGUMENT,
                     "mnb_shard_columns: bad rank/world");
        const int64_t base = n / world_size, extra = n % world_size;
        *col_count = base + (rank < extra ? 1 : 0);
        *col_begin = int64_t(rank) * base + std::min<int64_t>(rank, extra);
    });
}

int mnb_context_create(int device, mnb_context** out) {
    return guard([&] {
        auto* c = new mnb_context;
        try {
            init_context(c->ctx, device);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void mnb_last_parse_location(int64_t* line, int64_t* column) {
    if (line) *line = g_parse_line;
    if (column) *column = g_parse_column;
}

int mnb_mm_read_dims(const char* path, int64_t* rows, int64_t* cols) {
    return guard([&] {
        mnb::require(path && rows && cols, MNB_ERR_INVALID_ARGUMENT, "mnb_mm_read_dims: null argument");
        mnb::mm_dims(path, rows, cols);
    });
}

int mnb_mm_read(const char* path, void* out, int64_t rows, int64_t cols) {
    return guard([&] {
        mnb::require(path && out && rows >= 1 && cols >= 1, MNB_ERR_INVALID_ARGUMENT, "mnb_mm_read: bad argument");
        mnb::mm_read(path, static_cast<double*>(out), rows, cols);
    });
}

int mnb_mm_write(const char* path, const void* data, int64_t rows, int64_t cols) {
    return guard([&] {
        mnb::require(path && (data || rows * cols == 0) && rows >= 0 && cols >= 0, MNB_ERR_INVALID_ARGUMENT,
                     "mnb_mm_write: bad argument");
        mnb::mm_write(path, static_cast<const double*>(data), rows, cols);
    });
}

int mnb_generate_instance(int64_t m, int64_t n, double kappa, uint64_t stream_seed, void* A_out, void* b_out,
                          void* p_out) {
    return guard([&] {
        mnb::require(A_out && b_out && p_out, MNB_ERR_INVALID_ARGUMENT, "mnb_generate_instance: null output");
        mnb::generate_instance(m, n, kappa, stream_seed, static_cast<double*>(A_out), static_cast<double*>(b_out),
                               static_cast<double*>(p_out));
    });
}

int mnb_redistribute_plan(int64_t m, int64_t n_global, int world_size, int rank, int64_t* plan) {
    return guard([&] {
        mnb::require(world_size >= 1 && rank >= 0 && rank < world_size && m >= 1 && n_global >= 1 && plan,
                     MNB_ERR_INVALID_ARGUMENT, "mnb_redistribute_plan: bad arguments");
        mnb::redistribute_plan(m, n_global, world_size, rank, plan);
    });
}

int mnb_nccl_unique_id(void* out128) {
    return guard([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        nccl_ok(ncclGetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof id);
    });
}

int mnb_context_create_distributed(int device, int rank, int world_size, const void* nccl_unique_id, mnb_context** out) {
    return guard([&] {
        mnb::require(world_size >= 1 && rank >= 0 && rank < world_size, MNB_ERR_INVALID_ARGUMENT, "bad rank/world");
        auto* c = new mnb_context;
        try {
            init_context(c->ctx, device);
            c->ctx.rank = rank;
            c->ctx.world = world_size;
            ncclUniqueId id;
            std::memcpy(&id, nccl_unique_id, sizeof id);
            nccl_ok(ncclCommInitRank(&c->ctx.comm, world_size, id, rank), "ncclCommInitRank");
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void mnb_context_destroy(mnb_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->ctx.device);
    cudaStreamSynchronize(ctx->ctx.stream);
    delete ctx;
}

int mnb_context_set_stream(mnb_context* ctx, void* stream) {
    return guard([&] {
        auto& c = ctx->ctx;
        if (c.own_stream && c.stream) MNB_CUDA(cudaStreamDestroy(c.stream));
        c.stream = static_cast<cudaStream_t>(stream);
        c.own_stream = false;
        cublasSetStream(c.cublas, c.stream);
        cusolverDnSetStream(c.cusolver, c.stream);
    });
}

int mnb_set_matrix(mnb_context* ctx, int dtype, int64_t m, int64_t n_global, int64_t col_begin, int64_t n_local,
                   const void* A, int64_t lda, int location) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        mnb::require(dtype == MNB_C128 || dtype == MNB_F64, MNB_ERR_INVALID_ARGUMENT, "dtype must be C128 or F64");
        mnb::require(m >= 1 && n_global >= 1 && n_local >= 0 && col_begin >= 0 && col_begin + n_local <= n_global,
                     MNB_ERR_DIMENSION, "mnb_set_matrix: inconsistent dimensions");
        mnb::require(lda >= m, MNB_ERR_INVALID_ARGUMENT, "mnb_set_matrix: lda < m");
        c.slab_ready = false;
        if (c.distributed()) {
            int64_t b = 0, cnt = 0;
            mnb_shard_columns(n_global, c.world, c.rank, &b, &cnt);
            mnb::require(b == col_begin && cnt == n_local, MNB_ERR_DIMENSION,
                         "mnb_set_matrix: shard must follow mnb_shard_columns");
        }
        const size_t esz = dtype == MNB_F64 ? 8 : 16;
        // the fused pass streams columns with 16-byte bulk copies: a real A with odd m is promoted
        const bool promote = dtype == MNB_F64 && (m % 2);
        c.dtype = promote ? MNB_C128 : dtype;
        c.m = m;
        c.n_global = n_global;
        c.col_begin = col_begin;
        c.n_local = n_local;
        if (location == MNB_DEVICE && lda == m && !promote) {
            c.A = A;
            return;
        }
        const size_t out_esz = c.esz();
        void* dst = c.A_own.ensure(std::max<size_t>(size_t(m) * size_t(n_local) * out_esz, 16));
        c.pending_host = false;
        c.A_host = nullptr;
        if (location == MNB_HOST_ASYNC && !c.distributed() && !promote && n_local > 0) {
            cudaPointerAttributes attr{};
            const bool pinned = cudaPointerGetAttributes(&attr, A) == cudaSuccess && attr.type == cudaMemoryTypeHost;
            cudaGetLastError();
            if (pinned) {
                c.A = dst;
                c.A_host = A;
                c.host_lda = lda;
                c.pending_host = true;
                return;
            }
        }
        const auto kind = location == MNB_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        if (!promote) {
            MNB_CUDA(cudaMemcpy2DAsync(dst, size_t(m) * esz, A, size_t(lda) * esz, size_t(m) * esz, size_t(n_local), kind,
                                       c.stream));
        } else {
            // interleave (a, 0) on the device: copy the real values into the real slots
            mnb::require(lda == m, MNB_ERR_UNSUPPORTED, "real A with odd m requires lda == m");
            MNB_CUDA(cudaMemsetAsync(dst, 0, size_t(m) * size_t(n_local) * 16, c.stream));
            MNB_CUDA(cudaMemcpy2DAsync(dst, 16, A, 8, 8, size_t(m) * size_t(n_local), kind, c.stream));
        }
        MNB_CUDA(cudaStreamSynchronize(c.stream));
        c.A = dst;
    });
}

void mnb_solver_config_default(mnb_solver_config* cfg) {
    cfg->sketch_size = 0;
    cfg->alpha = 4.0;
    cfg->epsilon = 1e-6;
    cfg->seed = 42;
    cfg->sampling = MNB_WITHOUT_REPLACEMENT;
    cfg->capture_c = 0;
    cfg->lsq_max_iterations = 300;
}

int mnb_solve_randomized(mnb_context* ctx, const void* b, int b_location, const mnb_solver_config* cfg, void* x_out,
                         int x_location, void* c_out, mnb_solve_report* report) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        std::vector<double2> bh(size_t(c.m));
        if (b_location == MNB_DEVICE)
            MNB_CUDA(cudaMemcpy(bh.data(), b, size_t(c.m) * 16, cudaMemcpyDeviceToHost));
        else
            std::memcpy(bh.data(), b, size_t(c.m) * 16);
        const size_t nb = size_t(std::max<int64_t>(c.n_local, 1)) * 16;
        double2* x_dev = x_location == MNB_DEVICE ? static_cast<double2*>(x_out)
                                                  : static_cast<double2*>(c.vec_n[3].ensure(nb));
        double2* c_dev = nullptr;
        if (c_out) c_dev = x_location == MNB_DEVICE ? static_cast<double2*>(c_out)
                                                    : static_cast<double2*>(c.out_c.ensure(nb));
        mnb_solve_report rep{};
        mnb::solve_randomized(c, bh.data(), *cfg, x_dev, c_dev, rep);
        if (x_location != MNB_DEVICE && c.n_local) {
            copy_out(x_out, x_dev, size_t(c.n_local) * 16, MNB_HOST, c.stream);
            if (c_out) copy_out(c_out, c_dev, size_t(c.n_local) * 16, MNB_HOST, c.stream);
        }
        mnb::sync(c);
        if (report) *report = rep;
    });
}

int mnb_solve_classical(mnb_context* ctx, const void* b, int b_location, void* x_out, int x_location,
                        mnb_classical_report* report) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        std::vector<double2> bh(size_t(c.m));
        if (b_location == MNB_DEVICE)
            MNB_CUDA(cudaMemcpy(bh.data(), b, size_t(c.m) * 16, cudaMemcpyDeviceToHost));
        else
            std::memcpy(bh.data(), b, size_t(c.m) * 16);
        const size_t nb = size_t(std::max<int64_t>(c.n_local, 1)) * 16;
        double2* x_dev = x_location == MNB_DEVICE ? static_cast<double2*>(x_out)
                                                  : static_cast<double2*>(c.vec_n[3].ensure(nb));
        mnb_classical_report rep{};
        mnb::solve_classical(c, bh.data(), x_dev, rep);
        if (x_location != MNB_DEVICE && c.n_local) copy_out(x_out, x_dev, size_t(c.n_local) * 16, MNB_HOST, c.stream);
        mnb::sync(c);
        if (report) *report = rep;
    });
}

int mnb_solve_least_squares(mnb_context* ctx, const void* cvec, int c_location, const mnb_lsq_config* cfg, void* y_out,
                            double* residual_norms, mnb_lsq_solution* sol) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        ctx->ctx.make_resident();
        const double2* c_dev = static_cast<const double2*>(cvec);
        if (c_location != MNB_DEVICE) {
            double2* d = static_cast<double2*>(c.vec_n[2].ensure(size_t(std::max<int64_t>(c.n_local, 1)) * 16));
            MNB_CUDA(cudaMemcpyAsync(d, cvec, size_t(c.n_local) * 16, cudaMemcpyHostToDevice, c.stream));
            c_dev = d;
        }
        mnb_lsq_solution s{};
        mnb::solve_least_squares(c, c_dev, *cfg, static_cast<double2*>(y_out), residual_norms, s);
        if (sol) *sol = s;
    });
}

// ------------------------------------------------------------ SRFT ------
int mnb_srft_build(int64_t l, int64_t n, uint64_t stream_seed, int sampling, mnb_srft** out) {
    return guard([&] {
        auto* op = new mnb_srft;
        try {
            mnb::build_srft_host(op->host, l, n, stream_seed, sampling,
                                 [](size_t b) { return static_cast<unsigned char*>(std::malloc(b)); },
                                 [](unsigned char* p) { std::free(p); }, 0);
        } catch (...) {
            delete op;
            throw;
        }
        *out = op;
    });
}

int mnb_srft_from_fields(int64_t l, int64_t n, int sampling, const double* d, const int64_t* sample, const double* theta,
                         const double* theta_tilde, const int64_t* perm, const int64_t* perm_tilde, const double* zeta,
                         const double* zeta_tilde, mnb_srft** out) {
    return guard([&] {
        mnb::require(n >= 2 && l >= 1 && l <= n, MNB_ERR_INVALID_ARGUMENT, "srft_from_fields: need n >= 2, 1 <= l <= n");
        auto* op = new mnb_srft;
        auto& h = op->host;
        h.n = n;
        h.l = l;
        h.sampling = sampling;
        h.layout();
        h.blob = static_cast<unsigned char*>(std::malloc(h.total_bytes));
        h.release = [](unsigned char* p) { std::free(p); };
        std::memcpy(h.at<double>(h.off_d), d, size_t(n) * 16);
        std::memcpy(h.at<double>(h.off_zeta), zeta, size_t(n) * 16);
        std::memcpy(h.at<double>(h.off_zeta_tilde), zeta_tilde, size_t(n) * 16);
        std::memcpy(h.at<double>(h.off_theta), theta, size_t(n - 1) * 8);
        std::memcpy(h.at<double>(h.off_theta_tilde), theta_tilde, size_t(n - 1) * 8);
        std::memcpy(h.at<int64_t>(h.off_sample64), sample, size_t(l) * 8);
        int32_t* p = h.at<int32_t>(h.off_perm);
        int32_t* pt = h.at<int32_t>(h.off_perm_tilde);
        for (int64_t i = 0; i < n; ++i) {
            p[i] = int32_t(perm[i]);
            pt[i] = int32_t(perm_tilde[i]);
        }
        double* cs = h.at<double>(h.off_cssn);
        double* cst = h.at<double>(h.off_cssn_tilde);
        for (int64_t j = 0; j < n - 1; ++j) {  // finalize (src/srft.cpp:80-93)
            ::sincos(theta[j], &cs[2 * j + 1], &cs[2 * j]);
            ::sincos(theta_tilde[j], &cst[2 * j + 1], &cst[2 * j]);
        }
        cs[2 * (n - 1)] = cst[2 * (n - 1)] = 1.0;
        cs[2 * (n - 1) + 1] = cst[2 * (n - 1) + 1] = 0.0;
        h.derive();
        *out = op;
    });
}

void mnb_srft_destroy(mnb_srft* op) { delete op; }

int mnb_srft_dims(const mnb_srft* op, int64_t* l, int64_t* n) {
    *l = op->host.l;
    *n = op->host.n;
    return MNB_OK;
}

int mnb_srft_get_field(const mnb_srft* op, int field, void* out) {
    return guard([&] {
        const auto& h = op->host;
        const size_t n = size_t(h.n), l = size_t(h.l);
        auto unpack_cs = [&](size_t off, int which) {
            const double* cs = h.at<double>(off);
            double* o = static_cast<double*>(out);
            for (size_t j = 0; j + 1 < n; ++j) o[j] = cs[2 * j + which];
        };
        auto widen = [&](size_t off, size_t count) {
            const int32_t* p = h.at<int32_t>(off);
            int64_t* o = static_cast<int64_t*>(out);
            for (size_t i = 0; i < count; ++i) o[i] = p[i];
        };
        switch (field) {
            case MNB_FIELD_D: std::memcpy(out, h.at<double>(h.off_d), n * 16); break;
            case MNB_FIELD_ZETA: std::memcpy(out, h.at<double>(h.off_zeta), n * 16); break;
            case MNB_FIELD_ZETA_TILDE: std::memcpy(out, h.at<double>(h.off_zeta_tilde), n * 16); break;
            case MNB_FIELD_THETA: std::memcpy(out, h.at<double>(h.off_theta), (n - 1) * 8); break;
            case MNB_FIELD_THETA_TILDE: std::memcpy(out, h.at<double>(h.off_theta_tilde), (n - 1) * 8); break;
            case MNB_FIELD_COS_THETA: unpack_cs(h.off_cssn, 0); break;
            case MNB_FIELD_SIN_THETA: unpack_cs(h.off_cssn, 1); break;
            case MNB_FIELD_COS_THETA_TILDE: unpack_cs(h.off_cssn_tilde, 0); break;
            case MNB_FIELD_SIN_THETA_TILDE: unpack_cs(h.off_cssn_tilde, 1); break;
            case MNB_FIELD_PERM: widen(h.off_perm, n); break;
            case MNB_FIELD_PERM_TILDE: widen(h.off_perm_tilde, n); break;
            case MNB_FIELD_SAMPLE: std::memcpy(out, h.at<int64_t>(h.off_sample64), l * 8); break;
            default: throw mnb::Error(MNB_ERR_INVALID_ARGUMENT, "unknown SRFT field id");
        }
    });
}

static int srft_vec_op(mnb_context* ctx, const mnb_srft* op, const void* in, void* out, int which) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        const auto& h = op->host;
        const size_t n = size_t(h.n), l = size_t(h.l);
        const size_t nin = which == 2 ? l : n, nout = which == 1 ? l : n;
        mnb::SrftDev& dev = c.op_dev[2];
        mnb::upload_srft(c, h, dev);
        double2* din = static_cast<double2*>(c.vec_m[6].ensure(std::max(nin, n) * 16));
        double2* dout = static_cast<double2*>(c.vec_m[7].ensure(std::max(nout, n) * 16));
        MNB_CUDA(cudaMemcpyAsync(din, in, nin * 16, cudaMemcpyHostToDevice, c.stream));
        if (which == 2) mnb::srft_adjoint_vec(c, dev, din, dout);
        else mnb::srft_apply_vec(c, dev, din, dout, which == 0);
        MNB_CUDA(cudaMemcpyAsync(out, dout, nout * 16, cudaMemcpyDeviceToHost, c.stream));
        mnb::sync(c);
    });
}

int mnb_srft_apply_h(mnb_context* ctx, const mnb_srft* op, const void* x, void* y) { return srft_vec_op(ctx, op, x, y, 0); }
int mnb_srft_apply(mnb_context* ctx, const mnb_srft* op, const void* x, void* y) { return srft_vec_op(ctx, op, x, y, 1); }
int mnb_srft_apply_adjoint(mnb_context* ctx, const mnb_srft* op, const void* v, void* y) {
    return srft_vec_op(ctx, op, v, y, 2);
}

int mnb_srft_apply_to_columns(mnb_context* ctx, const mnb_srft* op, void* out, int out_location) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        ctx->ctx.make_resident();
        mnb::require(c.A != nullptr || c.n_local == 0, MNB_ERR_INVALID_ARGUMENT, "no problem matrix set");
        mnb::require(op->host.n == c.n_global, MNB_ERR_INVALID_ARGUMENT, "apply_to_columns: matrix must have n rows");
        mnb::SrftDev& dev = c.op_dev[2];
        mnb::upload_srft(c, op->host, dev);
        const size_t bytes = size_t(op->host.l) * size_t(c.m) * 16;
        double2* S = out_location == MNB_DEVICE ? static_cast<double2*>(out)
                                                : static_cast<double2*>(c.sk_S.ensure(bytes));
        c.slab_ready = false;  // the matrix may have changed in place since the last exchange
        mnb::sketch_matrix(c, dev, S, nullptr, nullptr);
        if (out_location != MNB_DEVICE) copy_out(out, S, bytes, MNB_HOST, c.stream);
        mnb::sync(c);
    });
}

int mnb_dft(mnb_context* ctx, int64_t n, void* x, int inverse) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        mnb::require(n >= 1, MNB_ERR_INVALID_ARGUMENT, "Fft: length must be positive");
        if (n == 1) return;
        double2* d = static_cast<double2*>(c.vec_m[6].ensure(size_t(n) * 16));
        MNB_CUDA(cudaMemcpyAsync(d, x, size_t(n) * 16, cudaMemcpyHostToDevice, c.stream));
        mnb::dft_vec(c, n, d, inverse != 0);
        MNB_CUDA(cudaMemcpyAsync(x, d, size_t(n) * 16, cudaMemcpyDeviceToHost, c.stream));
        mnb::sync(c);
    });
}

int mnb_apply_adjoint_matrix(mnb_context* ctx, const void* y, int y_location, void* x_out, int x_location,
                             void* ax_out) {
    return guard([&] {
        auto& c = ctx->ctx;
        MNB_CUDA(cudaSetDevice(c.device));
        c.make_resident();
        const size_t nb = size_t(std::max<int64_t>(c.n_local, 1)) * 16;
        double2* x_dev = x_location == MNB_DEVICE ? static_cast<double2*>(x_out)
                                                  : static_cast<double2*>(c.vec_n[3].ensure(nb));
        mnb::apply_adjoint_matrix(c, y, y_location == MNB_DEVICE, x_dev, static_cast<double2*>(ax_out));
        if (x_location != MNB_DEVICE && c.n_local) copy_out(x_out, x_dev, size_t(c.n_local) * 16, MNB_HOST, c.stream);
        mnb::sync(c);
    });
}

int mnb_bench_pcg_pass(mnb_context* ctx, int reps, double* ms_per_launch) {
    return guard([&] {
        MNB_CUDA(cudaSetDevice(ctx->ctx.device));
        ctx->ctx.make_resident();
        *ms_per_launch = mnb::bench_pcg_pass(ctx->ctx, std::max(1, reps));
    });
}

int mnb_chol_upper(mnb_context* ctx, void* G, int64_t m, double shift_factor, double rank_rows, double* status) {
    return guard([&] {
        auto& c = ctx->ctx;
        mnb::require(m >= 1 && G && status, MNB_ERR_INVALID_ARGUMENT, "mnb_chol_upper: bad arguments");
        MNB_CUDA(cudaSetDevice(c.device));
        const size_t bytes = size_t(m) * size_t(m) * 16;
        auto* Gd = static_cast<double2*>(c.gram.ensure(bytes));
        auto* st = static_cast<mnb::CholStatus*>(c.qr_status.ensure(sizeof(mnb::CholStatus) + sizeof(mnb::RefineStatus)));
        MNB_CUDA(cudaMemcpyAsync(Gd, G, bytes, cudaMemcpyHostToDevice, c.stream));
        MNB_CUDA(cudaEventRecord(c.event(60), c.stream));
        mnb::launch_chol_upper(Gd, m, m, shift_factor, rank_rows, st, c.num_sms, c.stream);
        MNB_CUDA(cudaEventRecord(c.event(61), c.stream));
        mnb::CholStatus h{};
        MNB_CUDA(cudaMemcpyAsync(G, Gd, bytes, cudaMemcpyDeviceToHost, c.stream));
        MNB_CUDA(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, c.stream));
        mnb::sync(c);
        status[0] = h.info;
        status[1] = h.deficient;
        status[2] = h.dmin;
        status[3] = h.dmax;
        status[4] = h.trace;
        status[5] = h.shift;
        float ms = 0.f;
        MNB_CUDA(cudaEventElapsedTime(&ms, c.event(60), c.event(61)));
        status[6] = ms;
    });
}

int mnb_trtri_upper(mnb_context* ctx, const void* R, int64_t m, void* X, double* xnorm2) {  // xnorm2: out2
    return guard([&] {
        auto& c = ctx->ctx;
        mnb::require(m >= 1 && R && X, MNB_ERR_INVALID_ARGUMENT, "mnb_trtri_upper: bad arguments");
        MNB_CUDA(cudaSetDevice(c.device));
        const size_t bytes = size_t(m) * size_t(m) * 16;
        auto* Rd = static_cast<double2*>(c.gram.ensure(bytes));
        auto* Xd = static_cast<double2*>(c.Rinv.ensure(bytes));
        auto* Wd = static_cast<double2*>(c.tri_work.ensure(bytes));
        auto* st = static_cast<mnb::CholStatus*>(c.qr_status.ensure(sizeof(mnb::CholStatus) + sizeof(mnb::RefineStatus)));
        MNB_CUDA(cudaMemcpyAsync(Rd, R, bytes, cudaMemcpyHostToDevice, c.stream));
        MNB_CUDA(cudaEventRecord(c.event(60), c.stream));
        mnb::launch_trtri_upper(Rd, m, m, Xd, Wd, st, c.num_sms, c.stream);
        MNB_CUDA(cudaEventRecord(c.event(61), c.stream));
        mnb::CholStatus h{};
        MNB_CUDA(cudaMemcpyAsync(X, Xd, bytes, cudaMemcpyDeviceToHost, c.stream));
        MNB_CUDA(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, c.stream));
        mnb::sync(c);
        if (xnorm2) {
            xnorm2[0] = h.xnorm2;
            float ms = 0.f;
            MNB_CUDA(cudaEventElapsedTime(&ms, c.event(60), c.event(61)));
            xnorm2[1] = ms;
        }
    });
}

int mnb_csne_solve(mnb_context* ctx, const void* S, int64_t l, int64_t m, const void* b, void* z, double* status) {
    return guard([&] {
        auto& c = ctx->ctx;
        mnb::require(m >= 1 && l >= m && S && b && z && status, MNB_ERR_INVALID_ARGUMENT, "mnb_csne_solve: bad arguments");
        MNB_CUDA(cudaSetDevice(c.device));
        mnb::csne_solve_host(c, static_cast<const double2*>(S), l, m, static_cast<const double2*>(b),
                             static_cast<double2*>(z), status);
    });
}

}  // extern "C"
