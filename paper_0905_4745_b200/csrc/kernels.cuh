// Launch interfaces of the sm_100a kernels (host-callable).
#pragma once

#include "common.cuh"

namespace mnb {

// ---------------------------------------------------------------- H stage
struct HStageArgs {
    // input element (r, k) = in[in_row0 + r + k*ld_in] (complex, or real promoted)
    const void* in = nullptr;
    int in_real = 0, in_conj = 0;
    int64_t ld_in = 0, in_row0 = 0;
    const int32_t* gather = nullptr;   // post-gather index i reads column gather[i]
    const double2* in_diag = nullptr;  // x <- x * diag[src]   (conj if in_diag_conj)
    int in_diag_conj = 0;
    const double2* cssn = nullptr;     // (cos theta_j, sin theta_j)
    const int32_t* halo = nullptr;     // per-chunk start index of the recurrence
    int adjoint = 0;
    double2* out = nullptr;
    int64_t ld_out = 0, out_row0 = 0;
    const int32_t* scatter = nullptr;  // output index o goes to column scatter[o]
    const double2* out_diag = nullptr; // y <- y * diag[dst]   (conj if out_diag_conj)
    int out_diag_conj = 0;
    int64_t rows = 0, n = 0, chunk = 0, nchunks = 0;
    int* nonfinite = nullptr;          // if set: flag any non-finite input entry (ProblemInstance::validate)
};
void launch_hstage(const HStageArgs& a, cudaStream_t stream);

// Sketch H stage (forward chain over row blocks, cp.async ring; k_hchain.cu).
struct HChainArgs {
    const void* in = nullptr;          // element (r, k) = in[in_row0 + r + k*ld_in]
    int in_real = 0, in_conj = 0;
    int64_t ld_in = 0, in_row0 = 0;
    const int32_t* gather = nullptr;   // step j reads column gather[j]
    const double2* params = nullptr;   // [n][3] = {cs_j, zin_j, zout_{j+1}} (build_chain_params)
    int has_zin = 0, has_zout = 0;
    double2 zout0 = {1.0, 0.0};        // output diagonal at index 0
    const int32_t* halo = nullptr;     // per-chunk start index
    double2* out = nullptr;
    int64_t ld_out = 0, out_row0 = 0;
    int64_t rows = 0, n = 0, chunk = 0, nchunks = 0, max_span = 0;
    int* nonfinite = nullptr;
    // blocked output for the four-step FFT (n = n1*n2): element (row, o) at
    // out + (row/8)*n*8 + ((o % n1)*n2 + o / n1)*8 + row%8; 0 = [n][ld_out] layout
    int64_t blk_n1 = 0, blk_n2 = 0;
};
void launch_hchain(const HChainArgs& a, int num_sms, cudaStream_t stream);
bool hchain_fits(int64_t max_span, int is_real);
void build_chain_params(const double2* cssn, const double2* zin, const int32_t* zin_index, const double2* zout,
                        int64_t n, double2* rec, cudaStream_t stream);

// Fused second H stage + FFT pass A (k_p2fa.cu): n = n1 x 1024, chain chunks of n1 (1024, 3072).
struct P2faArgs {
    const double2* x1 = nullptr;     // first-stage output, element (r, i) at x1[r + i * ld]
    int64_t ld = 0;
    const int32_t* gather = nullptr; // Pi: step j reads column gather[j]
    const double2* rec = nullptr;    // [n][3] {cs_j, -, d_{j+1}} (build_chain_params, zout = d)
    double2 zout0 = {1.0, 0.0};      // d_0
    const int32_t* halo = nullptr;   // per-chunk restart index (forward chain of Theta)
    const int32_t* halo_seg = nullptr; // restart index per (n1 / 2)-index sub-chunk (split row blocks)
    int64_t full_rb = 1 << 30;       // row blocks run whole; the rest run as two k1 segments
    int n1 = 1024;                   // chain chunk = k1 steps per row block
    const double2* carries = nullptr; // chain carries at the segment bounds [2048][ldc] (launch_p2fa_carries)
    int64_t ldc = 0;
    int sync_mask = 15;              // cluster barrier every sync_mask + 1 steps (power of two; 16 measured best)
    const double2* tw = nullptr;     // w_1024^q
    const double2* rec_t = nullptr;  // step-major {cs_j, d_{j+1}} [n1 s][1024 c] (build_p2fa_tables)
    const int32_t* idx_t = nullptr;  // step-major gather indices [n1 s][1024 c]
    const double2* z_t = nullptr;    // four-step twiddles w_n^{f k1} [n1 k1][1024 f] (build_p2fa_twiddles)
    double2* out = nullptr;          // pass A output, blocked [row block][f2][k1][8]
    int64_t rows = 0;                // multiple of 8
};
bool p2fa_supported(int64_t n, int64_t n1, int64_t n2, int64_t rows);
bool p2fa_chunk_ok(int64_t n1);  // chain chunk / pass-B lengths the fused path covers
void launch_p2fa(const P2faArgs& a, int num_sms, cudaStream_t stream);
// the restart prologues of launch_p2fa: carries[k * a.ldc + row] for the 1024 chunk ends (and the
// 1024 chunk midpoints when row blocks split); a.carries / a.ldc must point at this buffer
void launch_p2fa_carries(const P2faArgs& a, double2* carries, cudaStream_t stream);
void build_p2fa_tables(const double2* rec, const int32_t* gather, int n1, double2* rec_t, int32_t* idx_t,
                       cudaStream_t stream);
void build_p2fa_twiddles(const double2* hi, const double2* lo, int shift, int n1, double2* z_t, cudaStream_t stream);

// ---------------------------------------------------------------- FFT
enum FftOutMode { FFT_OUT_TWIDDLE = 0, FFT_OUT_SELECT = 1, FFT_OUT_NATURAL = 2 };

struct FftPassArgs {
    const double2* in = nullptr;
    int64_t ld_in = 0, in_row0 = 0;
    int64_t in_bstride = 0, in_istride = 1;  // column = b*in_bstride + idx*in_istride
    double2* out = nullptr;
    int64_t ld_out = 0, out_row0 = 0;
    int mode = FFT_OUT_NATURAL;
    int64_t out_fstride = 0, out_bstride = 0; // TWIDDLE: column = f*out_fstride + b*out_bstride
    int64_t nb = 1;                           // SELECT/NATURAL: frequency = b + nb*f
    const int32_t* sel = nullptr;             // SELECT: frequency -> output slot (or -1)
    double scale = 1.0;
    const double2* tw = nullptr;              // w_N^q, q < N   (forward sign)
    const double2* tw4_hi = nullptr;          // four-step twiddle w_n^e = hi[e>>sh] * lo[e & mask]
    const double2* tw4_lo = nullptr;
    int tw4_shift = 0;
    int64_t n_total = 1;
    int N = 1;
    int nradix = 0;
    int radix[10] = {0};
    int E = 1;                                // elements per thread
    int Rb = 1;                               // rows per CTA
    int64_t rows = 0;                         // rows in this block (masking)
    int64_t batches = 1;                      // grid.y
    int inverse = 0;
    // blocked four-step layout (sketch): input tile of unit (rbk, b) at in + (rbk*batches + b)*N*Rb,
    // TWIDDLE output at out + ((rbk*N + f)*batches + b)*Rb + r (rows padded to a multiple of Rb)
    int blocked = 0;
    int num_sms = 148;
};
void launch_fft_pass(const FftPassArgs& a, cudaStream_t stream);
// Blocked pass B with N = 1024, pruned to the sampled frequencies: per batch f2 the CSR list
// off[f2] .. off[f2+1] of (f1, slot) pairs in ent (forward, SELECT semantics of FftPassArgs).
void launch_fft1024_select(const FftPassArgs& a, const int32_t* off, const int32_t* ent, cudaStream_t stream);
// Pass B pruned to the sampled frequencies, plain [n][Ms] layout, N = 16 U (U <= 128).
// Returns false (nothing launched) when the shape is not covered.
bool launch_fft_select_pruned(const FftPassArgs& a, const int32_t* off, const int32_t* ent, int num_sms,
                              cudaStream_t stream);
// Pruned pass B over the blocked layout of the fused H stage + pass A for N = 3072
// (n = 3 * 2^20); false when the shape is not covered.
bool launch_fft_select_blocked(const FftPassArgs& a, const int32_t* off, const int32_t* ent, int num_sms,
                               cudaStream_t stream);
// O(N^2) fallback for lengths without a 2^a 3^b factorisation (N <= 4096).
void launch_dft_direct(const FftPassArgs& a, cudaStream_t stream);
// Largest per-thread element count E (and radix plan) for an in-smem length N;
// returns false when N has prime factors other than 2 and 3.
bool plan_radices(int N, int& E, int* radix, int& nradix);

// ---------------------------------------------------------------- misc
// chain restart points for chunks of `chunk` indices (forward and adjoint chains)
void launch_chain_halos(const double2* cssn, int64_t n, int64_t chunk, int64_t nchunks, int32_t* fwd, int32_t* adj,
                        cudaStream_t stream);
// zero the strictly lower triangle of an m x m column-major matrix
void launch_zero_lower(double2* A, int64_t m, cudaStream_t stream);
// y = S^H z for the column-major l x m sketch (deterministic, no cuBLAS handle: safe beside
// library work on another stream)
void launch_sketch_adjoint_gemv(const double2* S, int64_t l, int64_t m, const double2* z, double2* y,
                                cudaStream_t stream);
// out = in + 0i
void launch_real_to_complex(const double* in, double2* out, int64_t count, cudaStream_t stream);
// x <- conj(x)
void launch_conj_inplace(double2* x, int64_t count, cudaStream_t stream);
// r = c, t = 0, x = 0 (x may be null), red_scal[0..3] = [||c||^2, 0, 0, 0]; part: `parts` doubles of scratch
void launch_cg_init_vectors(const double2* c, int64_t n, double2* r, double2* t, double2* x, double* part, int parts,
                            double* red_scal, cudaStream_t stream);
// A_jj += shift (real), m x m column-major
void launch_add_diagonal(double2* A, int64_t m, double shift, cudaStream_t stream);
// power steps on Q1^H Q1 - I (cholqr_r): v <- v / *nrm, a <- v ; and a <- a - v, v <- a
void launch_unit_copy(double2* v, double2* a, int64_t m, const double* nrm, cudaStream_t stream);
void launch_sub_copy(double2* a, double2* v, int64_t m, cudaStream_t stream);
// out[0] = max_{i<=j} |A_ij - delta_ij| over the upper triangle (deterministic)
void launch_max_offset_from_identity(const double2* A, int64_t m, double* out, cudaStream_t stream);
void launch_copy_dups(double2* S, int64_t ldS, int64_t row0, int64_t rows, const int32_t* dups, int64_t ndups,
                      cudaStream_t stream);
void launch_scatter_add_sample(const double2* v, int64_t l, const int32_t* sample, int with_replacement,
                               double2* w, int64_t n, cudaStream_t stream);

}  // namespace mnb
