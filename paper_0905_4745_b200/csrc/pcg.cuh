// Fused preconditioned-CG kernels: interfaces and device-resident state.
#pragma once

#include "common.cuh"

namespace mnb {

// Device-resident CG state of solve_least_squares (src/lsq.cpp:77-111).
struct CgState {
    double gg;        // ||g_k||^2 (lsq.cpp:81)
    double gg_prev;   // copy of gg taken by upd1 for upd2's beta
    double alpha;     // step of the last update; consumed by the next pass as alpha_prev
    double rr;        // estimate of ||r_{k+1}||^2 from exact <r_k,t_k>, ||t_k||^2
    double rr0;       // ||c||^2
    double floor2;    // 1e-28 ||c||^2 (lsq.cpp:82)
    double tau;
    double dup;       // max multiplicity (lsq.cpp:70)
    double excess;    // dup * gg at the last convergence test
    double rr_final;  // exact ||r||^2 of the returned iterate (finalize)
    double xx_final;  // ||x||^2 of x = sum_k alpha_k t_k (finalize; the Step-5 vector)
    long long iterations;
    long long max_iterations;
    int done;
    int converged;
    int stop_qq0;
    int pad;
};

enum PcgMode {
    PCG_CG = 0,    // t = A^H w; s = A t; lagged r update; store t in place
    PCG_INIT = 1,  // t given (= c); s = A c; r <- c; t <- 0; qq = ||c||^2
    PCG_APPLY = 2, // t = A^H w stored to tout (x = A^H y); s = A t; qq = ||t||^2
};

struct PcgPassArgs {
    const void* A = nullptr;  // column-major m x n (lda == m), complex or real
    int is_real = 0;
    int64_t m = 0, n = 0;
    const double2* w = nullptr;    // m
    const double2* tin = nullptr;  // n (INIT: c; CG: t_{k-1})
    double2* tout = nullptr;       // n (CG: same as tin; APPLY: x)
    double2* r = nullptr;          // n
    double2* x = nullptr;          // n or null: x += alpha_prev t_prev (CG), x = 0 (INIT)
    const CgState* state = nullptr;
    double2* part_s = nullptr;     // [grid][m]
    double* part_scal = nullptr;   // [grid][4]: qq, Re<r,t>, ||r||^2, -
    int mode = PCG_CG;
};

struct PcgPlan {
    int grid = 0;
    int G = 1, EPL = 1, K = 1, stages = 4;  // warps per group, rows per thread, columns per batch
    int64_t stage_cols = 1;                  // columns per shared-memory stage (groups x K)
    int64_t per_cta = 1;                     // contiguous columns per CTA
    size_t smem = 0;
};
PcgPlan plan_pcg_pass(int64_t m, int64_t n, int is_real, int num_sms);
void launch_pcg_pass(const PcgPassArgs& a, const PcgPlan& plan, cudaStream_t stream);

// s = sum of part_s, scalars = sum of part_scal (fixed order) -> red = [s (m complex), qq, rt, rr, 0]
void launch_pcg_reduce(const double2* part_s, const double* part_scal, int parts, int64_t m, double* red,
                       const CgState* state, cudaStream_t stream);
// upd1: alpha = gg/qq; u += alpha dir; g -= alpha Rinv^H s; dir_old = dir; part_gg
void launch_pcg_upd1(const double* red, const double2* Rinv, int64_t m, double2* u, double2* g, const double2* dir,
                     double2* dir_old, double* part_gg, CgState* state, double* residual_norms, int init,
                     cudaStream_t stream, double2* ax = nullptr);
// upd2: gg' = sum part_gg; convergence; dir = g + beta dir_old; w = Rinv dir
void launch_pcg_upd2(const double* part_gg, int parts_gg, const double2* Rinv_rows, int64_t m, const double2* g,
                     const double2* dir_old, double2* dir, double2* w, CgState* state, int init,
                     cudaStream_t stream);
int pcg_upd_blocks(int64_t m);
// r <- r - alpha t, x <- x + alpha t (pending updates), ||r||^2 -> rr_final, ||x||^2 -> xx_final
void launch_pcg_finalize(double2* r, const double2* t, double2* x, int64_t n, CgState* state, double* scratch,
                         cudaStream_t stream);
// y = Rinv u (upper triangular, row layout)
void launch_trmv_rows(const double2* Rinv_rows, int64_t m, const double2* u, double2* y, cudaStream_t stream);
// out[j*ld_out + i] = in[i*ld_in + j] (complex transpose, m x m)
void launch_transpose(const double2* in, int64_t rows, int64_t cols, int64_t ld_in, double2* out, int64_t ld_out,
                      cudaStream_t stream);
void launch_init_state(CgState* st, double tau, double dup, long long max_it, cudaStream_t stream);

// The whole CG loop as one persistent cooperative kernel (k_pcg_small.cu) for L2-resident A.
constexpr int64_t kSmallMaxM = 256;
struct SmallCgArgs {
    const void* A = nullptr;  // column-major m x n (lda == m)
    int is_real = 0;
    int64_t m = 0, n = 0;
    const double2* Rinv = nullptr;       // m x m upper, column layout
    const double2* Rinv_rows = nullptr;  // the same, row layout
    double2 *u = nullptr, *g = nullptr, *dir = nullptr, *dir_old = nullptr, *w = nullptr, *ax = nullptr;  // m
    double2 *r = nullptr, *t = nullptr, *x = nullptr;                                                    // n
    double2* part_s = nullptr;    // [grid][m]
    double* part_scal = nullptr;  // [grid][4]
    double2* s = nullptr;         // m
    double* part_gg = nullptr;    // [grid]
    CgState* st = nullptr;
    double* residual_norms = nullptr;
};
bool pcg_small_eligible(int64_t m, int64_t n, int is_real);
int pcg_small_grid(int64_t m, int64_t n, int num_sms);
void launch_pcg_small(const SmallCgArgs& a, int grid, cudaStream_t stream);
// one iteration's reduce + gradient + direction phases as one cooperative launch (A, n, x unused)
int pcg_update_grid(int64_t m, int num_sms);
void launch_pcg_update(const SmallCgArgs& a, int parts, int grid, cudaStream_t stream);

}  // namespace mnb
