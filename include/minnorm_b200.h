/* minnorm_b200.h -- C ABI of the B200-native randomized minimal-norm hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch / Eigen
 * types.  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).  A matrix is always the
 * reference's layout: column-major complex<double> (interleaved re,im; 16 B),
 * `A` is m x n with m < n, lda >= m (include/minnorm/types.hpp:10,
 * SPEC.md:461).  A real float64 A (BASELINE config 5) is an extension.
 *
 * All functions return an MNB_* status; the message of the last failure on
 * the calling thread is available from mnb_last_error().  The status codes
 * map one-to-one onto the reference's exceptions
 * (include/minnorm/errors.hpp:10-49) so a C++ shim can rethrow them and keep
 * the CLI exit-code map of tools/minnorm_main.cpp:29-35.
 */
#ifndef MINNORM_B200_H
#define MINNORM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define MNB_OK 0
#define MNB_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument (lsq.cpp:47-55, srft.cpp:97-98) */
#define MNB_ERR_CONFIG 2           /* minnorm::ConfigError (errors.hpp:10-13)            */
#define MNB_ERR_DIMENSION 3        /* minnorm::DimensionError (errors.hpp:16-19)         */
#define MNB_ERR_RANK_DEFICIENCY 4  /* minnorm::RankDeficiencyError (errors.hpp:22-31)    */
#define MNB_ERR_CUDA 5
#define MNB_ERR_NCCL 6
#define MNB_ERR_UNSUPPORTED 7      /* e.g. an FFT length this build has no kernel for   */
#define MNB_ERR_OUT_OF_MEMORY 8
#define MNB_ERR_INTERNAL 9
#define MNB_ERR_PARSE 10           /* minnorm::ParseError (errors.hpp:34-49)             */

/* ---- enums --------------------------------------------------------------- */
#define MNB_C128 0 /* complex<double> */
#define MNB_F64 1  /* double (real A; config 5) */
#define MNB_HOST 0
#define MNB_DEVICE 1
#define MNB_HOST_ASYNC 2 /* mnb_set_matrix: pinned host A, copied by the next solve in row slabs that
                            overlap its sketches (caller keeps A alive until that call returns) */
#define MNB_WITHOUT_REPLACEMENT 0 /* RandomStream::Sampling (rng.hpp:18) */
#define MNB_WITH_REPLACEMENT 1

/* ---- errors / version ---------------------------------------------------- */
const char* mnb_last_error(void);
/* RankDeficiencyError::deficient_columns() of the last MNB_ERR_RANK_DEFICIENCY. */
int64_t mnb_last_deficient_columns(void);
const char* mnb_version(void);

/* ParseError::line() / column() of the last MNB_ERR_PARSE (1-based, 0 when unknown). */
void mnb_last_parse_location(int64_t* line, int64_t* column);

/* ---- dense complex Matrix Market files (host only; no GPU needed) ----------
 * The reference front end's file format (include/minnorm/matrix_market.hpp,
 * src/matrix_market.cpp:65-130): "%%MatrixMarket matrix array complex general",
 * comments, "rows cols", then one "re im" pair per line in column-major order.
 * Malformed input -> MNB_ERR_PARSE with the reference's line / column. */
/* read_matrix_market, step 1: the size line only. */
int mnb_mm_read_dims(const char* path, int64_t* rows, int64_t* cols);
/* read_matrix_market (matrix_market.cpp:65-102), step 2: the entries into out
 * (rows*cols complex<double>, column-major); rows/cols as returned by step 1. */
int mnb_mm_read(const char* path, void* out, int64_t rows, int64_t cols);
/* write_matrix_market (matrix_market.cpp:113-130): 17 significant digits. */
int mnb_mm_write(const char* path, const void* data, int64_t rows, int64_t cols);

/* generate_instance(m, n, kappa, RandomStream(stream_seed)) (include/minnorm/bench.hpp;
 * src/bench.cpp:46-74), host only: A = U diag(sigma) V^H (m x n column-major complex),
 * b = A p_true (m), p_true = V w (n).  Same substreams (21/22/23) and draw order as the
 * reference; values agree to rounding (the products are summed in a different order).
 * Bad sizes -> MNB_ERR_DIMENSION (the CLI maps the reference's invalid_argument there). */
int mnb_generate_instance(int64_t m, int64_t n, double kappa, uint64_t stream_seed, void* A_out, void* b_out,
                          void* p_out);

/* ---- context (one per GPU / per rank) ------------------------------------ */
typedef struct mnb_context mnb_context;

int mnb_context_create(int device, mnb_context** out);
/* Column-sharded multi-GPU context: one process per GPU, NCCL communicator
 * built from a 128-byte ncclUniqueId that rank 0 created with
 * mnb_nccl_unique_id() and the launcher broadcast.  world_size 1 is allowed and
 * takes the distributed code path (all-to-all, allgather, per-iteration
 * allreduce) over a one-rank communicator. */
int mnb_nccl_unique_id(void* out128);
int mnb_context_create_distributed(int device, int rank, int world_size, const void* nccl_unique_id,
                                   mnb_context** out);
void mnb_context_destroy(mnb_context* ctx);
/* Run on the caller's CUDA stream (cudaStream_t) instead of the context's own. */
int mnb_context_set_stream(mnb_context* ctx, void* cuda_stream);
/* Column partition used by every multi-GPU entry point (pure host logic). */
int mnb_shard_columns(int64_t n, int world_size, int rank, int64_t* col_begin, int64_t* col_count);
/* The distributed sketch's one all-to-all (column shards -> row blocks; pure host logic, the
 * table the CUDA path itself follows).  For every peer h = 0..world_size-1 of `rank`, six
 * entries at plan[6h..6h+5]:
 *   send_row0, send_rows  rows of A that rank h owns (mnb_shard_columns(m, world, h));
 *   send_offset           element offset of block h in the pack buffer: block h is
 *                         A[send_row0 : +send_rows, this rank's columns], column-major, ld send_rows;
 *   recv_col0, recv_cols  columns rank h owns (mnb_shard_columns(n_global, world, h));
 *   recv_offset           element offset (recv_col0 * my_rows) in this rank's row block, which is
 *                         my_rows x n_global, column-major, ld my_rows.
 * Replaces the reference's serial column loop over B = A^* (src/srft.cpp:147-153) being cut
 * into row blocks; there is no reference counterpart (single process). */
int mnb_redistribute_plan(int64_t m, int64_t n_global, int world_size, int rank, int64_t* plan);

/* The problem matrix A (ProblemInstance::A, include/minnorm/solver.hpp:14-24):
 * this rank's column shard A[:, col_begin : col_begin+n_local], column-major
 * with leading dimension lda >= m.  location MNB_DEVICE borrows the pointer
 * (caller keeps it alive; requires lda == m; the library's work is ordered on
 * the context's stream only, so the caller completes -- or orders through
 * mnb_context_set_stream -- whatever produces A), MNB_HOST copies it to the GPU,
 * MNB_HOST_ASYNC (single GPU, page-locked host memory; otherwise as MNB_HOST)
 * defers the copy: mnb_solve_randomized streams A in row slabs and sketches
 * each slab as it lands, and any other call first completes the copy. */
int mnb_set_matrix(mnb_context* ctx, int dtype, int64_t m, int64_t n_global, int64_t col_begin,
                   int64_t n_local, const void* A, int64_t lda, int location);

/* ---- the solver (include/minnorm/solver.hpp:26-63) ------------------------ */
typedef struct {
    int64_t sketch_size;        /* SolverConfig::sketch_size; 0 = default 4m            */
    double alpha;               /* SolverConfig::alpha (4.0)                             */
    double epsilon;             /* SolverConfig::epsilon (1e-6)                          */
    uint64_t seed;              /* SolverConfig::seed (42, rng.hpp:20)                   */
    int32_t sampling;           /* SolverConfig::sampling (without replacement)          */
    int32_t capture_c;          /* SolverConfig::capture_c                              */
    int64_t lsq_max_iterations; /* SolverConfig::lsq_max_iterations (300)               */
} mnb_solver_config;

typedef struct {
    double step_seconds[5];  /* SolveReport::step_seconds (device events per step)      */
    double c_norm_ratio;     /* SolveReport::c_norm_ratio                               */
    double residual_norm;    /* SolveReport::residual_norm = ||A x - b||                */
    int64_t lsq_iterations;  /* SolveReport::lsq_iterations                             */
    int32_t lsq_converged;   /* SolveReport::lsq_converged                              */
    int32_t qr_path;         /* extension: sketch QR used, S in bits 0-3, E in bits 4-7:
                                0 CholeskyQR2, 1 shifted CholeskyQR3, 2 Householder,
                                3 one Cholesky pass (E, preconditioner only),
                                4 one Cholesky pass + corrected seminormal Step 2 (S),
                                5 shifted two-pass Cholesky (E, preconditioner only),
                                6 shifted two-pass Cholesky + corrected seminormal Step 2 (S) */
    int64_t sketch_size;     /* SolveReport::sketch_size                                */
    double lsq_tau;          /* SolveReport::lsq_tau                                    */
    /* ---- extensions (not in the reference report) ---- */
    double lsq_achieved_excess;  /* LsqSolution::achieved_excess (lsq.hpp:21)           */
    double param_seconds;        /* host SRFT parameter generation (both operators)     */
    double total_seconds;        /* whole solve, host wall clock                        */
    double sketch_seconds[2];    /* device time of sketch S (step 1) and E (step 4)     */
    double redistribute_seconds; /* all-to-all of A into row blocks (multi-GPU)         */
    double qr_seconds[2];        /* device time of the two QRs                          */
    double pcg_seconds;          /* device time of the CG loop                          */
    double pcg_pass_ms_sum;      /* summed device time of the fused A(A^H w) passes     */
    int64_t pcg_pass_launches;   /* number of fused-pass launches timed above           */
    double sketch_kernel_ms[4];  /* summed device time per sketch kernel family:
                                    [0] H stage 1, [1] H stage 2, [2] FFT pass A, [3] FFT pass B */
    int64_t kernel_launches;     /* kernels this solve launched (own kernels only)      */
    int64_t world_size;
} mnb_solve_report;

void mnb_solver_config_default(mnb_solver_config* cfg);

/* solve_randomized(const ProblemInstance&, const SolverConfig&)
 * (include/minnorm/solver.hpp:55; src/solver.cpp:50-128).
 * b: m complex values; x_out: this rank's n_local complex values of x;
 * c_out: optional (NULL) n_local values of the Step-3 vector c. */
int mnb_solve_randomized(mnb_context* ctx, const void* b, int b_location, const mnb_solver_config* cfg,
                         void* x_out, int x_location, void* c_out, mnb_solve_report* report);

/* ---- the classical solver (include/minnorm/solver.hpp:59; src/solver.cpp:130-146) ----
 * The deterministic O(m^2 n) baseline the paper compares against (t0 of Tables 1-4).
 * On the GPU: Gram G = A A^H (tensor-core ZHERK; one allreduce across ranks), R1 = chol(G),
 * and the corrected seminormal equations z_{k+1} = z_k + G^{-1}(b - A A^H z_k), x = A^H z,
 * each correction one fused pass over A; accepted once ||b - A x|| is at the rounding level
 * of A x.  When u cond(A)^2 is not small (the Cholesky fails or the corrections do not
 * contract) it falls back to Householder QR of A^H (cuSOLVER Xgeqrf + Xunmqr; one GPU),
 * the reference's algorithm without the column pivoting (complex A; real A takes path 0 only).
 * b: m complex values; x_out: this rank's n_local complex values.                        */
typedef struct {
    int32_t path;          /* 0 Gram + corrected seminormal equations, 1 Householder QR of A^H */
    int32_t refinements;   /* corrections taken on path 0                                       */
    double residual_norm;  /* ||A x - b||                                                        */
    double seconds;        /* wall time of the call                                              */
} mnb_classical_report;

int mnb_solve_classical(mnb_context* ctx, const void* b, int b_location, void* x_out, int x_location,
                        mnb_classical_report* report);

/* ---- the least-squares subsolver (include/minnorm/lsq.hpp:12-40) --------- */
typedef struct {
    int64_t sketch_size;    /* LsqConfig::sketch_size                                   */
    double tau;             /* LsqConfig::tau                                           */
    int64_t max_iterations; /* LsqConfig::max_iterations                               */
    uint64_t stream_seed;   /* seed of LsqConfig::stream (RandomStream::seed())         */
    int32_t sampling;       /* LsqConfig::sampling                                      */
    int32_t reserved0;
} mnb_lsq_config;

typedef struct {
    double achieved_excess; /* LsqSolution::achieved_excess */
    int64_t iterations;     /* LsqSolution::iterations      */
    int32_t converged;      /* LsqSolution::converged       */
    int32_t reserved0;
} mnb_lsq_solution;

/* solve_least_squares(B, c, cfg) with B = A^H of the context matrix
 * (src/lsq.cpp:43-113; the only B the solver ever passes, src/solver.cpp:112).
 * c: n_local complex; y_out: m complex (host); residual_norms: optional array
 * of max_iterations+1 doubles (LsqSolution::residual_norms). */
int mnb_solve_least_squares(mnb_context* ctx, const void* c, int c_location, const mnb_lsq_config* cfg,
                            void* y_out, double* residual_norms, mnb_lsq_solution* sol);

/* ---- the SRFT operator (include/minnorm/srft.hpp:21-65) ------------------- */
typedef struct mnb_srft mnb_srft;

/* build_srft(l, n, RandomStream(stream_seed), sampling) (src/srft.cpp:95-113):
 * host-side, bit-identical parameters to the reference RandomStream. */
int mnb_srft_build(int64_t l, int64_t n, uint64_t stream_seed, int sampling, mnb_srft** out);
/* An operator from explicit fields (tests: trivial / hand-built operators;
 * tests/test_support.hpp:110-126).  Complex arrays interleaved. */
int mnb_srft_from_fields(int64_t l, int64_t n, int sampling, const double* d, const int64_t* sample,
                         const double* theta, const double* theta_tilde, const int64_t* perm,
                         const int64_t* perm_tilde, const double* zeta, const double* zeta_tilde,
                         mnb_srft** out);
void mnb_srft_destroy(mnb_srft* op);
/* Copy a parameter field out (field ids as MNB_FIELD_*). */
#define MNB_FIELD_D 0
#define MNB_FIELD_ZETA 1
#define MNB_FIELD_ZETA_TILDE 2
#define MNB_FIELD_THETA 3
#define MNB_FIELD_THETA_TILDE 4
#define MNB_FIELD_COS_THETA 5
#define MNB_FIELD_SIN_THETA 6
#define MNB_FIELD_COS_THETA_TILDE 7
#define MNB_FIELD_SIN_THETA_TILDE 8
#define MNB_FIELD_PERM 9
#define MNB_FIELD_PERM_TILDE 10
#define MNB_FIELD_SAMPLE 11
int mnb_srft_get_field(const mnb_srft* op, int field, void* out);
int mnb_srft_dims(const mnb_srft* op, int64_t* l, int64_t* n);

/* SrftOperator::apply_h / apply / apply_adjoint (src/srft.cpp:115-145) on the GPU,
 * host vectors in and out (tests and single-vector use). */
int mnb_srft_apply_h(mnb_context* ctx, const mnb_srft* op, const void* x, void* y);
int mnb_srft_apply(mnb_context* ctx, const mnb_srft* op, const void* x, void* y);
int mnb_srft_apply_adjoint(mnb_context* ctx, const mnb_srft* op, const void* v, void* y);
/* SrftOperator::apply_to_columns(B) with B = A^H of the context matrix
 * (src/srft.cpp:147-153 as called at src/solver.cpp:81 and src/lsq.cpp:56):
 * out = l x m column-major (complex), on host or device.  Multi-GPU: includes
 * the all-to-all into row blocks; every rank receives the full sketch. */
int mnb_srft_apply_to_columns(mnb_context* ctx, const mnb_srft* op, void* out, int out_location);

/* Unitary DFT (src/fft.cpp:90-110; include/minnorm/fft.hpp:12) of a host vector. */
int mnb_dft(mnb_context* ctx, int64_t n, void* x, int inverse);

/* ---- benchmarking hooks (device-resident, CUDA-event timed) -------------- */
/* Times `reps` launches of the fused PCG pass s = A(A^H w), qq = ||A^H w||^2
 * over the context matrix; returns the mean per-launch milliseconds. */
/* Step 5 of solve_randomized as a standalone product (src/solver.cpp:118-125): x = A^H y for
 * this rank's columns, and (ax_out != NULL) A x = A A^H y summed over ranks -- one fused pass
 * over A (the PCG pass kernel in its apply mode).  y: m complex (host or device);
 * x_out: n_local complex; ax_out: m complex (host).                                          */
int mnb_apply_adjoint_matrix(mnb_context* ctx, const void* y, int y_location, void* x_out, int x_location,
                             void* ax_out);

int mnb_bench_pcg_pass(mnb_context* ctx, int reps, double* ms_per_launch);

/* ---- the sketch-QR building blocks (hand-written kernels, csrc/k_cholqr.cu) ------------------
 * The reference factors both sketches with Eigen::HouseholderQR (src/solver.cpp:86,
 * src/lsq.cpp:58) and applies R by triangular solves (src/solver.cpp:93-96, src/lsq.cpp:71-73).
 * Here R comes from the Gram matrix; these entries expose the three device stages on host
 * arrays (column-major complex128) so they can be checked on their own.
 *
 * mnb_chol_upper: in-place upper Cholesky G = R^H R of the Hermitian m x m matrix whose upper
 * triangle is in G (the strictly lower triangle is zeroed); shift_factor * trace(G) is added to
 * the diagonal first (0 = none).  status[7] = {info (LAPACK potrf convention), deficient (the rank
 * rule of src/solver.cpp:25-33 with `rows` = rank_rows), min R_jj, max R_jj, trace(G), shift,
 * kernel milliseconds (CUDA events)}.
 * mnb_trtri_upper: X = R^{-1} for upper-triangular R; out2 (optional) = {||X||_F^2, kernel ms}.
 * mnb_csne_solve: Step 2's z = Q R^{-H} b (src/solver.cpp:93-96) for the l x m sketch S from the
 * corrected seminormal equations (Gram, Cholesky, inverse and refinement all on the device);
 * status[4] = {accepted, corrections, ||b - S^H z||, ||z||}.                                   */
int mnb_chol_upper(mnb_context* ctx, void* G, int64_t m, double shift_factor, double rank_rows, double* status);
int mnb_trtri_upper(mnb_context* ctx, const void* R, int64_t m, void* X, double* out2);
int mnb_csne_solve(mnb_context* ctx, const void* S, int64_t l, int64_t m, const void* b, void* z, double* status);

#ifdef __cplusplus
}
#endif

#endif /* MINNORM_B200_H */
