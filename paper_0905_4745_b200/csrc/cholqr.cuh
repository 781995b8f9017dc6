// Hand-written sm_100a kernels for the sketch QRs (src/solver.cpp:86-96, src/lsq.cpp:58-64):
// blocked Cholesky of the Gram matrix, the triangular inverse, and the device-resident
// refinement loops on top of them (Step 2's corrected seminormal equations, the one-pass
// preconditioner's orthogonality check).  Every decision the host used to take between library
// calls (pivot failure, diagonal ratio, rank rule, refinement stop) is taken on the device and
// reported in one status record, so a sketch QR is a handful of launches and one host read.
#pragma once

#include "common.cuh"

namespace mnb {

// Filled by launch_chol_upper (device memory; 64 bytes).
struct CholStatus {
    int info;          // 0, or 1 + index of the first non-positive pivot (LAPACK potrf convention)
    int deficient;     // rank rule: # of R_jj < rank_rows * eps * max R_jj (or == 0); valid when info == 0
    double dmin, dmax; // min / max of the diagonal of R
    double trace;      // trace(G) before the shift = ||R||_F^2 = ||S||_F^2
    double shift;      // the diagonal shift that was applied (shift_factor * trace)
    double xnorm2;     // ||R^{-1}||_F^2 (launch_trtri_upper)
    double pad[2];
};

// Filled by launch_sketch_refine (device memory).
struct RefineStatus {
    int accepted;      // CSNE: residual floor at the rounding level; PRECOND: one pass accepted
    int iterations;    // corrections / power steps taken
    int frobenius_ok;  // PRECOND: accepted on the Frobenius bound alone
    int pad0;
    double best;       // CSNE: smallest ||b - S^H z||;  PRECOND: ||D v|| of the last power step
    double nz_best;    // CSNE: ||z|| at that iterate
    double thr;        // CSNE: 2 sqrt(l) u ||S||_F ; PRECOND: u ||R1||_F^2 ||R1^{-1}||_F^2
    double resid[8];   // CSNE: ||b - S^H z_k|| per correction (trace / tests)
};

// grid sizes for the cooperative launches (one CTA per SM at most)
int chol_grid(int64_t m, int num_sms);

// In-place upper Cholesky G = R^H R of the Hermitian m x m matrix whose upper triangle is in G
// (column-major, leading dimension ld); the strictly lower triangle is zeroed.  A real shift
// shift_factor * trace(G) is added to the diagonal first (shifted CholeskyQR; 0 = none).
// rank_rows: the `rows` of the reference's rank rule (src/solver.cpp:25-33, src/lsq.cpp:18-27).
void launch_chol_upper(double2* G, int64_t m, int64_t ld, double shift_factor, double rank_rows, CholStatus* st,
                       int num_sms, cudaStream_t stream);

// X = R^{-1} for the upper-triangular m x m R (leading dimension ldr); X and the workspace W are
// m x m with leading dimension m; X's strictly lower triangle comes out zero.  st->xnorm2 (optional).
// gate_on_chol: st is the record of the Cholesky that produced R; skip when that failed (info, or
// a diagonal ratio with u ratio^2 > 1e-3) -- the host will redo the factorization anyway.
void launch_trtri_upper(const double2* R, int64_t ldr, int64_t m, double2* X, double2* W, CholStatus* st,
                        int num_sms, cudaStream_t stream, bool gate_on_chol = false);

// st->deficient = the rank rule's count on the diagonal of R = R2 R1 (two upper Cholesky factors)
void launch_diag_product_rank(const double2* R2, int64_t ld2, const double2* R1, int64_t ld1, int64_t m, double rows,
                              CholStatus* st, cudaStream_t stream);

enum RefineMode { REFINE_CSNE = 0, REFINE_PRECOND = 1 };
struct RefineArgs {
    int mode = REFINE_CSNE;
    const double2* S = nullptr;  // l x m sketch, column-major, leading dimension l
    int64_t l = 0, m = 0;
    const double2* X = nullptr;  // R1^{-1} (m x m upper, lower zero, leading dimension m)
    const CholStatus* chol = nullptr;
    const double2* b = nullptr;  // CSNE: right-hand side (m).  PRECOND: start vector of the power steps (m)
    double2* z = nullptr;        // CSNE: solution (l).  PRECOND: scratch (l)
    double2* v0 = nullptr;       // scratch m-vectors
    double2* v1 = nullptr;
    double2* v2 = nullptr;
    double* part = nullptr;      // scratch: at least l / 32 + 2 + grid doubles
    RefineStatus* st = nullptr;
    int power_steps = 10;
    int two_norm_check = 1;
};
void launch_sketch_refine(const RefineArgs& a, int num_sms, cudaStream_t stream);

}  // namespace mnb
