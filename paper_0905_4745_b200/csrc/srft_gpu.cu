// The SRFT on the GPU: sketch T·A^H (SrftOperator::apply_to_columns,
// src/srft.cpp:147-153), single-vector apply / apply_adjoint
// (src/srft.cpp:115-145) and the unitary DFT (src/fft.cpp:90-110).
//
// Sketch data flow for a slab of rows (all column-major, one column = the
// slab's rows contiguous):
//   P1  hstage: x1[:, i] = zeta[i] * Chain~( zeta~[p~[i]] * conj(A[:, p~[i]]) )   (H right half)
//   P2  hstage: x2[:, i] = d[i]    * Chain ( x1[:, p[i]] )                        (H left half, D)
//   FA  fft:    length-n2 DFTs over k2 of x2[:, k1 + n1 k2], twiddle w_n^{f2 k1} -> x1[:, f2 n1 + k1]
//   FB  fft:    length-n1 DFTs over k1, keep sampled f = f2 + n2 f1, scale n^{-1/2} -> S
// (n <= 2048: one FFT launch does the whole transform and the sampling.)
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cstring>
#include "context.cuh"

namespace mnb {

namespace {

void fill_twiddles(DevBuf& buf, int64_t N, int64_t count, int64_t step, cudaStream_t stream) {
    // buf[q] = exp(-2 pi i (q*step mod N) / N), computed in long double, rounded once.
    std::vector<double> h(size_t(2 * count));
    const long double two_pi = 6.283185307179586476925286766559L;
    for (int64_t q = 0; q < count; ++q) {
        const int64_t e = (q * step) % N;
        const long double ang = two_pi * (long double)e / (long double)N;
        h[size_t(2 * q)] = double(cosl(ang));
        h[size_t(2 * q + 1)] = double(-sinl(ang));
    }
    buf.ensure(size_t(count) * 16);
    MNB_CUDA(cudaMemcpyAsync(buf.p, h.data(), size_t(count) * 16, cudaMemcpyHostToDevice, stream));
    MNB_CUDA(cudaStreamSynchronize(stream));
}

bool smooth(int64_t N) {
    int E, r[10], nr;
    return N <= 1 || (N <= 8192 && plan_radices(int(N), E, r, nr));
}

void make_len_plan(FftLenPlan& p, int64_t N, cudaStream_t stream) {
    p.N = int(N);
    p.direct = !plan_radices(int(N), p.E, p.radix, p.nradix);
    fill_twiddles(p.tw, N, N, 1, stream);
}

// a blocked tile pass keeps 8 rows x N (+ half exchange) in shared memory, <= 512 threads
bool fft_tile_fits(int N, int E) { return size_t(N) * 12 * 16 + 16 <= size_t(227 * 1024) && 8 * N / E <= 512; }

int rows_per_cta(const FftLenPlan& p) {
    int rb = p.N <= 1024 ? 8 : 4;  // (8 rows at N = 1536 measured slower: one CTA per SM)
    while (rb > 1 && rb * p.N / std::max(p.E, 1) > 512) rb >>= 1;
    return rb;
}

FftPassArgs base_args(const FftLenPlan& p) {
    FftPassArgs a;
    a.N = p.N;
    a.E = p.E;
    a.nradix = p.nradix;
    for (int i = 0; i < p.nradix; ++i) a.radix[i] = p.radix[i];
    a.tw = p.tw.as<double2>();
    return a;
}

void run_fft(Context& ctx, const FftLenPlan& p, FftPassArgs a) {
    if (p.direct) launch_dft_direct(a, ctx.stream);
    else launch_fft_pass(a, ctx.stream);
    ctx.launches += 1;
}

// Kernel timing without host syncs: the event pair is resolved (summed into
// *acc) by Context::resolve_timers() at the end of the solve, so launches
// queue back to back and other streams can overlap them.
struct EventTimer {
    Context& ctx;
    double* acc;
    cudaEvent_t e0 = nullptr;
    EventTimer(Context& c, double* a, size_t /*slot*/) : ctx(c), acc(a) {
        if (acc) {
            e0 = ctx.timer_event();
            MNB_CUDA(cudaEventRecord(e0, ctx.stream));
        }
    }
    void stop() {
        if (acc) {
            cudaEvent_t e1 = ctx.timer_event();
            MNB_CUDA(cudaEventRecord(e1, ctx.stream));
            ctx.timers.push_back({e0, e1, acc});
        }
    }
};


// Length-n DFT of `rows` rows: in (col-major, ld_in) -> out.  SELECT keeps the
// sampled frequencies (out[slot + (out_row0 + r) * ld_out]); NATURAL writes
// all of them (out[(out_row0 + r) + f * ld_out]).  Scaled by n^{-1/2}.
void fft_rows(Context& ctx, int64_t n, const double2* in, int64_t ld_in, int64_t rows, double2* tmp, int64_t ld_tmp,
              double2* out, int64_t ld_out, int64_t out_row0, bool select, const int32_t* sel, bool inverse,
              double* ms_a, double* ms_b, const int32_t* fb_csr = nullptr) {
    FftPlan& P = ctx.fft_plan(n);
    const double scale = 1.0 / std::sqrt(double(n));
    auto rb = [&](const FftLenPlan& lp) { return rows == 1 ? 1 : rows_per_cta(lp); };
    if (P.single) {
        FftPassArgs a = base_args(P.A);
        a.in = in;
        a.ld_in = ld_in;
        a.in_bstride = 0;
        a.in_istride = 1;
        a.out = out;
        a.ld_out = ld_out;
        a.out_row0 = out_row0;
        a.mode = select ? FFT_OUT_SELECT : FFT_OUT_NATURAL;
        a.nb = 1;
        a.sel = sel;
        a.scale = scale;
        a.Rb = rb(P.A);
        a.rows = rows;
        a.batches = 1;
        a.inverse = inverse;
        EventTimer t(ctx, ms_a, 2);
        run_fft(ctx, P.A, a);
        t.stop();
        return;
    }
    {
        FftPassArgs a = base_args(P.A);
        a.in = in;
        a.ld_in = ld_in;
        a.in_bstride = 1;
        a.in_istride = P.n1;
        a.out = tmp;
        a.ld_out = ld_tmp;
        a.mode = FFT_OUT_TWIDDLE;
        a.out_fstride = P.n1;
        a.out_bstride = 1;
        a.tw4_hi = P.tw4_hi.as<double2>();
        a.tw4_lo = P.tw4_lo.as<double2>();
        a.tw4_shift = P.tw4_shift;
        a.n_total = n;
        a.Rb = rb(P.A);
        a.rows = rows;
        a.batches = P.n1;
        a.inverse = inverse;
        EventTimer t(ctx, ms_a, 2);
        run_fft(ctx, P.A, a);
        t.stop();
    }
    {
        FftPassArgs a = base_args(P.B);
        a.in = tmp;
        a.ld_in = ld_tmp;
        a.in_bstride = P.n1;
        a.in_istride = 1;
        a.out = out;
        a.ld_out = ld_out;
        a.out_row0 = out_row0;
        a.mode = select ? FFT_OUT_SELECT : FFT_OUT_NATURAL;
        a.nb = P.n2;
        a.sel = sel;
        a.scale = scale;
        a.Rb = rb(P.B);
        a.rows = rows;
        a.batches = P.n2;
        a.inverse = inverse;
        a.num_sms = ctx.num_sms;
        EventTimer t(ctx, ms_b, 3);
        // sketch: only the sampled frequencies are kept -> pruned pass B when the shape allows
        const bool pruned = select && fb_csr && rows > 1 && !P.B.direct &&
                            launch_fft_select_pruned(a, fb_csr, fb_csr + P.n2 + 1, ctx.num_sms, ctx.stream);
        if (pruned) ctx.launches += 1;
        else run_fft(ctx, P.B, a);
        t.stop();
    }
}

// Four-step DFT of `rows` rows held in the blocked layout of the sketch
// (see HChainArgs::blk_n1): pass A (length n2, twiddled) -> tmp (blocked for
// pass B), pass B (length n1) keeps the sampled frequencies -> out.
// a_done: pass A already ran (fused into the H stage, k_p2fa.cu) and its output is `in`.
void fft_rows_blocked(Context& ctx, int64_t n, const double2* in, int64_t rows, double2* tmp, double2* out,
                      int64_t ld_out, int64_t out_row0, const int32_t* sel, const int32_t* fb_csr, double* ms_a,
                      double* ms_b, bool a_done = false) {
    FftPlan& P = ctx.fft_plan(n);
    if (a_done) tmp = const_cast<double2*>(in);
    else {
        FftPassArgs a = base_args(P.A);
        a.in = in;
        a.out = tmp;
        a.mode = FFT_OUT_TWIDDLE;
        a.blocked = 1;
        a.num_sms = ctx.num_sms;
        a.tw4_hi = P.tw4_hi.as<double2>();
        a.tw4_lo = P.tw4_lo.as<double2>();
        a.tw4_shift = P.tw4_shift;
        a.n_total = n;
        a.Rb = fft_tile_fits(P.A.N, P.A.E) ? 8 : std::min(4, rows_per_cta(P.A));
        a.rows = rows;
        a.batches = P.n1;
        EventTimer t(ctx, ms_a, 2);
        launch_fft_pass(a, ctx.stream);
        ctx.launches += 1;
        t.stop();
    }
    {
        FftPassArgs a = base_args(P.B);
        a.in = tmp;
        a.out = out;
        a.ld_out = ld_out;
        a.out_row0 = out_row0;
        a.mode = FFT_OUT_SELECT;
        a.blocked = 1;
        a.num_sms = ctx.num_sms;
        a.nb = P.n2;
        a.sel = sel;
        a.scale = 1.0 / std::sqrt(double(n));
        a.Rb = fft_tile_fits(P.B.N, P.B.E) ? 8 : std::min(4, rows_per_cta(P.B));
        a.rows = rows;
        a.batches = P.n2;
        EventTimer t(ctx, ms_b, 3);
        const bool pruned = fb_csr && P.B.N == 1024 && !P.B.direct && a.Rb == 8;
        if (pruned) launch_fft1024_select(a, fb_csr, fb_csr + P.n2 + 1, ctx.stream);
        else if (!(a_done && fb_csr && launch_fft_select_blocked(a, fb_csr, fb_csr + P.n2 + 1, ctx.num_sms, ctx.stream)))
            launch_fft_pass(a, ctx.stream);
        ctx.launches += 1;
        t.stop();
    }
}
}  // namespace

FftPlan& Context::fft_plan(int64_t n) {
    auto it = fft_plans.find(n);
    if (it != fft_plans.end()) return *it->second;
    auto plan = std::make_unique<FftPlan>();
    FftPlan& P = *plan;
    P.n = n;
    if (n <= 2048 || (n <= 4096 && !smooth(n))) {
        P.single = true;
        P.n1 = 1;
        P.n2 = n;
        make_len_plan(P.A, n, stream);
    } else {
        // n = n1 * n2 with both factors smooth and <= 2048, as balanced as possible -- except
        // where the fused H stage + pass A (k_p2fa.cu) applies: n = n1 x 1024 with n1 = 128 ... 1024
        // or 3072 (c3: 128 x 1024, c5: 3072 x 1024)
        int64_t best = 0;
        const bool fused_split = p2fa && n % 1024 == 0 && p2fa_chunk_ok(n / 1024) && !std::getenv("MNB_FFT_BALANCED");
        if (fused_split) best = 1024;
        for (int64_t n2 = 2; n2 <= 2048 && !fused_split; ++n2) {
            if (n % n2) continue;
            const int64_t n1 = n / n2;
            if (n1 > 2048 || !smooth(n1) || !smooth(n2)) continue;
            if (!best || std::llabs(n1 - n2) < std::llabs(n / best - best)) best = n2;
        }
        require(best != 0, MNB_ERR_UNSUPPORTED,
                "FFT length " + std::to_string(n) + " is not supported on the GPU (needs n <= 4096, or n = n1*n2 "
                "with n1, n2 <= 2048 of the form 2^a 3^b)");
        P.single = false;
        P.n2 = best;
        P.n1 = n / best;
        make_len_plan(P.A, P.n2, stream);
        make_len_plan(P.B, P.n1, stream);
        int shift = 0;
        while ((int64_t(1) << (2 * shift)) < n) ++shift;
        P.tw4_shift = shift;
        const int64_t lo = int64_t(1) << shift, hi = (n + lo - 1) / lo;
        fill_twiddles(P.tw4_lo, n, lo, 1, stream);
        fill_twiddles(P.tw4_hi, n, hi, lo, stream);
    }
    fft_plans[n] = std::move(plan);
    return P;
}

// Device tables of the sketch's first H stage (needs perm~, cssn~, zeta~, zeta on the device).
static void build_tables_first(Context& ctx, const SrftHost& op, SrftDev& dev) {
    const int64_t n = op.n;
    double2* rec1 = static_cast<double2*>(dev.chain_rec[0].ensure(size_t(n) * 48));
    build_chain_params(dev.at<double2>(op.off_cssn_tilde), dev.at<double2>(op.off_zeta_tilde),
                       dev.at<int32_t>(op.off_perm_tilde), dev.at<double2>(op.off_zeta), n, rec1, ctx.stream);
    ctx.launches += 1;
}

static void build_tables_rest(Context& ctx, const SrftHost& op, SrftDev& dev);

void upload_srft(Context& ctx, const SrftHost& op, SrftDev& dev) {
    dev.host = &op;
    dev.blob.ensure(op.device_bytes);
    MNB_CUDA(cudaMemcpyAsync(dev.blob.p, op.blob, op.device_bytes, cudaMemcpyHostToDevice, ctx.stream));
    build_tables_first(ctx, op, dev);
    build_tables_rest(ctx, op, dev);
}

// Staged upload (SrftStage, host_srft.hpp): the groups of the first H stage go out as soon as
// the host has them; the rest follows on `side` (a copy stream) while that stage runs.
void upload_srft_first(Context& ctx, const SrftHost& op, SrftDev& dev) {
    dev.host = &op;
    dev.blob.ensure(op.device_bytes);
    unsigned char* d = static_cast<unsigned char*>(dev.blob.p);
    auto copy = [&](size_t b, size_t e) {
        MNB_CUDA(cudaMemcpyAsync(d + b, op.blob + b, e - b, cudaMemcpyHostToDevice, ctx.stream));
    };
    const size_t nc4 = size_t(op.ch.nchunks) * 4;
    copy(op.off_zeta, op.off_cssn);            // zeta, zeta~
    copy(op.off_cssn_tilde, op.off_perm);      // cos/sin(theta~)
    copy(op.off_perm_tilde, op.off_sel);       // perm~
    copy(op.off_halo + nc4, op.off_halo + 2 * nc4);      // restart points of the Theta~ chain: fwd~
    copy(op.off_halo + 3 * nc4, op.off_halo + 4 * nc4);  // adj~
    build_tables_first(ctx, op, dev);
}

void upload_srft_rest(Context& ctx, const SrftHost& op, SrftDev& dev, cudaStream_t side, cudaEvent_t landed) {
    unsigned char* d = static_cast<unsigned char*>(dev.blob.p);
    auto copy = [&](size_t b, size_t e) {
        MNB_CUDA(cudaMemcpyAsync(d + b, op.blob + b, e - b, cudaMemcpyHostToDevice, side));
    };
    const size_t nc4 = size_t(op.ch.nchunks) * 4;
    copy(op.off_d, op.off_zeta);                // d
    copy(op.off_cssn, op.off_cssn_tilde);       // cos/sin(theta)
    copy(op.off_perm, op.off_perm_tilde);       // perm
    copy(op.off_sel, op.off_halo + nc4);        // sel, fwd
    copy(op.off_halo + 2 * nc4, op.off_halo + 3 * nc4);  // adj
    copy(op.off_sample, op.device_bytes);       // sample
    MNB_CUDA(cudaEventRecord(landed, side));
    MNB_CUDA(cudaStreamWaitEvent(ctx.stream, landed, 0));
    build_tables_rest(ctx, op, dev);
}

static void build_tables_rest(Context& ctx, const SrftHost& op, SrftDev& dev) {
    const FftPlan& P = ctx.fft_plan(op.n);
    const int64_t n2 = P.single ? 0 : P.n2;
    // staging: [dups][csr offsets (n2 + 1)][(f1, slot) pairs (<= 2 l)]
    const size_t n_dups = op.dups.size(), n_csr = n2 ? size_t(n2 + 1) + 2 * size_t(op.l) : 0;
    if (dev.stage_free) MNB_CUDA(cudaEventSynchronize(dev.stage_free));  // previous upload out of the stage
    else MNB_CUDA(cudaEventCreateWithFlags(&dev.stage_free, cudaEventDisableTiming));
    int32_t* stage = static_cast<int32_t*>(dev.stage.ensure(std::max<size_t>(16, (n_dups + n_csr) * 4)));
    dev.ndups = int64_t(n_dups / 2);
    if (dev.ndups) {
        std::memcpy(stage, op.dups.data(), n_dups * 4);
        dev.dups.ensure(n_dups * 4);
        MNB_CUDA(cudaMemcpyAsync(dev.dups.p, stage, n_dups * 4, cudaMemcpyHostToDevice, ctx.stream));
    }
    // per-step records of the second sketch H stage (k_hchain.cu)
    const int64_t n = op.n;
    double2* rec2 = static_cast<double2*>(dev.chain_rec[1].ensure(size_t(n) * 48));
    build_chain_params(dev.at<double2>(op.off_cssn), nullptr, nullptr, dev.at<double2>(op.off_d), n, rec2, ctx.stream);
    ctx.launches += 1;
    // step-major tables of the fused second H stage + FFT pass A (k_p2fa.cu)
    if (ctx.p2fa && !P.single && p2fa_supported(n, P.n1, P.n2, 8)) {
        const int n1 = int(P.n1);
        build_p2fa_tables(rec2, dev.at<int32_t>(op.off_perm), n1,
                          static_cast<double2*>(dev.p2fa_rec.ensure(size_t(n) * 32)),
                          static_cast<int32_t*>(dev.p2fa_idx.ensure(size_t(n) * 4)), ctx.stream);
        // restart points of the chain chunks (n1 indices: one per k2) and of their halves
        // (the optional k1 segments): [fwd 1024][adj 1024][fwd 2048][adj 2048]
        int32_t* hs = static_cast<int32_t*>(dev.p2fa_halo.ensure(size_t(6 * 1024) * 4));
        launch_chain_halos(dev.at<double2>(op.off_cssn), n, n1, 1024, hs, hs + 1024, ctx.stream);
        launch_chain_halos(dev.at<double2>(op.off_cssn), n, n1 / 2, 2048, hs + 2048, hs + 4096, ctx.stream);
        ctx.launches += 3;
    }
    // fine restart points for single-vector H stages (apply / apply_adjoint of one vector)
    dev.vec_chunk = 32;
    dev.vec_nchunks = (n + dev.vec_chunk - 1) / dev.vec_chunk;
    {
        int32_t* vh = static_cast<int32_t*>(dev.vec_halo.ensure(size_t(4 * dev.vec_nchunks) * 4));
        const int64_t vc = dev.vec_nchunks;
        launch_chain_halos(dev.at<double2>(op.off_cssn), n, dev.vec_chunk, vc, vh, vh + 2 * vc, ctx.stream);
        launch_chain_halos(dev.at<double2>(op.off_cssn_tilde), n, dev.vec_chunk, vc, vh + vc, vh + 3 * vc, ctx.stream);
        ctx.launches += 2;
    }
    // kept frequencies grouped by f2 = F mod n2 for the pruned pass B (first occurrence of each F;
    // repeated samples are copied afterwards, launch_copy_dups)
    dev.fb_n2 = 0;
    if (n2) {
        const int64_t* s64 = op.at<int64_t>(op.off_sample64);
        const int32_t* sel = op.at<int32_t>(op.off_sel);
        int32_t* csr = stage + n_dups;
        std::memset(csr, 0, n_csr * 4);
        int32_t* off = csr;
        for (int64_t j = 0; j < op.l; ++j)
            if (sel[s64[j]] == int32_t(j)) ++off[s64[j] % n2 + 1];
        for (int64_t f2 = 0; f2 < n2; ++f2) off[f2 + 1] += off[f2];
        std::vector<int32_t> pos(off, off + n2);
        int32_t* ent = csr + n2 + 1;
        for (int64_t j = 0; j < op.l; ++j) {
            const int64_t F = s64[j];
            if (sel[F] != int32_t(j)) continue;
            const int32_t p = pos[size_t(F % n2)]++;
            ent[2 * p] = int32_t(F / n2);
            ent[2 * p + 1] = int32_t(j);
        }
        // within each f2, order the entries by f1 mod 16 (the pruned pass B loops over that
        // residue with a compile-time register index); stable, so ties keep the sample order
        for (int64_t f2 = 0; f2 < n2; ++f2) {
            int32_t* e = ent + 2 * off[f2];
            const int32_t cnt = off[f2 + 1] - off[f2];
            std::vector<std::pair<int32_t, int32_t>> v(static_cast<size_t>(cnt));
            for (int32_t i = 0; i < cnt; ++i) v[size_t(i)] = {e[2 * i], e[2 * i + 1]};
            std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return (x.first & 15) < (y.first & 15); });
            for (int32_t i = 0; i < cnt; ++i) {
                e[2 * i] = v[size_t(i)].first;
                e[2 * i + 1] = v[size_t(i)].second;
            }
        }
        dev.fb_csr.ensure(n_csr * 4);
        MNB_CUDA(cudaMemcpyAsync(dev.fb_csr.p, csr, n_csr * 4, cudaMemcpyHostToDevice, ctx.stream));
        dev.fb_n2 = n2;
    }
    MNB_CUDA(cudaEventRecord(dev.stage_free, ctx.stream));
}

// single vectors: the operator's fine 64-index chunks (more threads than rows x 1024-chunks)
static HStageArgs vec_chain_args(const SrftDev& op, bool tilde, bool adjoint) {
    const SrftHost& h = *op.host;
    HStageArgs a;
    a.cssn = op.at<double2>(tilde ? h.off_cssn_tilde : h.off_cssn);
    const int64_t nc = op.vec_nchunks;
    a.halo = op.vec_halo.as<int32_t>() + (adjoint ? 2 * nc : 0) + (tilde ? nc : 0);
    a.adjoint = adjoint ? 1 : 0;
    a.n = h.n;
    a.chunk = op.vec_chunk;
    a.nchunks = nc;
    return a;
}

static HStageArgs chain_args(const SrftDev& op, bool tilde, bool adjoint) {
    const SrftHost& h = *op.host;
    HStageArgs a;
    a.cssn = op.at<double2>(tilde ? h.off_cssn_tilde : h.off_cssn);
    const int32_t* halo = op.at<int32_t>(h.off_halo);
    const int64_t nc = h.ch.nchunks;
    a.halo = halo + (adjoint ? 2 * nc : 0) + (tilde ? nc : 0);
    a.adjoint = adjoint ? 1 : 0;
    a.n = h.n;
    a.chunk = h.ch.chunk;
    a.nchunks = nc;
    return a;
}

void sketch_block(Context& ctx, const SrftDev& op, const void* Ablk, int is_real, int64_t lda, int64_t row0,
                  int64_t rows, double2* out, int64_t ldo, int64_t out_row0, double* kernel_ms) {
    const SrftHost& h = *op.host;
    const int64_t n = h.n;
    ctx.fft_plan(n);
    // slab height: two n-column intermediates per slab row
    // (cached per shape: cudaMemGetInfo is a driver round trip, kept off the per-solve path)
    auto& sc = ctx.slab_cache;
    if (!(sc.n == n && sc.rows == rows && sc.l == h.l && sc.m == ctx.m)) {
        size_t free_b = 0, total_b = 0;
        MNB_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const size_t have = ctx.ws_x1.bytes + ctx.ws_x2.bytes + free_b;
        // keep room for what the solve allocates after the first sketch: the second
        // sketch E (l x m), the CholeskyQR2 copy (l x m), R, R', Gram, R'^{-1} twice (m x m), the second operator
        const size_t mm = size_t(ctx.m), ll = size_t(h.l);
        const size_t reserve = (size_t(2) << 30) + 40 * ll * mm + 128 * mm * mm + 2 * (h.device_bytes + 96 * size_t(n));
        const size_t budget = have > 2 * reserve ? have - reserve : have / 2;
        int64_t ms = std::min<int64_t>(rows, int64_t(budget / (size_t(32) * size_t(n))));
        if (ms < rows) ms = std::max<int64_t>(8, ms & ~int64_t(7));
        // the fused H + pass A runs one 8-row block per cluster pair: slabs of whole pair rounds
        // (c5: 840-row slabs = 105 blocks = 2 rounds on 74 pairs; 592 rows = 1 round)
        const FftPlan& fp0 = ctx.fft_plan(n);
        const int64_t round_rows = 8 * int64_t(ctx.num_sms / 2);
        if (ms < rows && ctx.p2fa && !fp0.single && p2fa_supported(n, fp0.n1, fp0.n2, 8) && ms >= round_rows)
            ms = ms / round_rows * round_rows;
        // MNB_SLAB_ROWS: force a smaller slab (tests of the multi-slab path at small m)
        if (const char* e = std::getenv("MNB_SLAB_ROWS"))
            if (const int64_t f = std::atoll(e); f > 0) ms = std::min<int64_t>(ms, std::max<int64_t>(8, f & ~int64_t(7)));
        sc = {n, rows, h.l, ctx.m, std::max<int64_t>(1, std::min<int64_t>(ms, rows))};
        if (std::getenv("MNB_TRACE"))
            std::fprintf(stderr, "[mnb] sketch slab: %lld of %lld rows (free %.1f GiB, budget %.1f GiB)\n",
                         (long long)sc.Ms, (long long)rows, double(free_b) / (1 << 30), double(budget) / (1 << 30));
    }
    const int64_t Ms = sc.Ms;
    const int64_t Mp = (Ms + 7) & ~int64_t(7);  // blocked layouts pad the slab to whole 8-row blocks
    double2* x1 = static_cast<double2*>(ctx.ws_x1.ensure(size_t(Mp) * size_t(n) * 16));
    double2* x2 = static_cast<double2*>(ctx.ws_x2.ensure(size_t(Mp) * size_t(n) * 16));
    const FftPlan& FP = ctx.fft_plan(n);
    // Four-step FFT with both passes' tiles (8 rows x N) in shared memory: P2 writes x2 in
    // the blocked layout pass A reads as contiguous tiles, pass A writes the one pass B reads.
    // (for longer passes, e.g. 1536 x 2048 at n = 3*2^20, the blocked layout read through 4-row
    // halves measured slower than the plain [n][Ms] layout: keep the latter there)
    const double scale = 1.0 / std::sqrt(double(n));

    for (int64_t s0 = 0; s0 < rows; s0 += Ms) {
        const int64_t rs = std::min(Ms, rows - s0);
        {  // P1: Z~, Pi~, Theta~, Z   (src/srft.cpp:52-55)
            EventTimer t(ctx, kernel_ms ? &kernel_ms[0] : nullptr, 0);
            if (hchain_fits(h.span_first, is_real)) {
                HChainArgs a;
                a.in = Ablk;
                a.in_real = is_real;
                a.in_conj = 1;  // column of B = A^H is conj(row of A)
                a.ld_in = lda;
                a.in_row0 = row0 + s0;
                a.gather = op.at<int32_t>(h.off_perm_tilde);
                a.params = op.chain_rec[0].as<double2>();
                a.has_zin = 1;
                a.has_zout = 1;
                a.zout0 = h.at<double2>(h.off_zeta)[0];
                a.halo = op.at<int32_t>(h.off_halo) + h.ch.nchunks;  // forward chain of Theta~
                a.out = x1;
                a.ld_out = Ms;
                a.rows = rs;
                a.n = n;
                a.chunk = h.ch.chunk;
                a.nchunks = h.ch.nchunks;
                a.max_span = h.span_first;
                a.nonfinite = ctx.nonfinite;
                launch_hchain(a, ctx.num_sms, ctx.stream);
            } else {
                HStageArgs a = chain_args(op, true, false);
                a.in = Ablk;
                a.in_real = is_real;
                a.in_conj = 1;
                a.ld_in = lda;
                a.in_row0 = row0 + s0;
                a.nonfinite = ctx.nonfinite;
                a.gather = op.at<int32_t>(h.off_perm_tilde);
                a.in_diag = op.at<double2>(h.off_zeta_tilde);
                a.out = x1;
                a.ld_out = Ms;
                a.out_diag = op.at<double2>(h.off_zeta);
                a.rows = rs;
                launch_hstage(a, ctx.stream);
            }
            ctx.launches += 1;
            t.stop();
        }
        // staged operator (SrftStage): its other half is uploaded now, behind the first H stage
        if (ctx.after_first_stage) {
            auto hook = std::move(ctx.after_first_stage);
            ctx.after_first_stage = nullptr;
            hook();
        }
        const bool chained = hchain_fits(h.max_span, is_real);
        const bool blocked = chained && !FP.single && !FP.A.direct && !FP.B.direct &&
                             fft_tile_fits(FP.A.N, FP.A.E) && fft_tile_fits(FP.B.N, FP.B.E);
        // P2 fused with FFT pass A (k_p2fa.cu) when the shape allows: x2 never goes to HBM
        const bool fused = chained && ctx.p2fa && op.p2fa_rec.p && !FP.single && p2fa_supported(n, FP.n1, FP.n2, rs);
        if (fused) {
            EventTimer t(ctx, kernel_ms ? &kernel_ms[1] : nullptr, 1);
            P2faArgs a;
            a.x1 = x1;
            a.ld = Ms;
            a.gather = op.at<int32_t>(h.off_perm);
            a.rec = op.chain_rec[1].as<double2>();
            a.zout0 = h.at<double2>(h.off_d)[0];
            a.halo = op.p2fa_halo.as<int32_t>();  // forward chain of Theta, chunks of n1
            a.tw = FP.A.tw.as<double2>();
            if (!FP.p2fa_z.p) {
                FftPlan& fp = ctx.fft_plan(n);
                build_p2fa_twiddles(fp.tw4_hi.as<double2>(), fp.tw4_lo.as<double2>(), fp.tw4_shift, int(fp.n1),
                                    static_cast<double2*>(fp.p2fa_z.ensure(size_t(n) * 16)), ctx.stream);
            }
            a.n1 = int(FP.n1);
            if (const char* e = std::getenv("MNB_P2FA_SYNC")) a.sync_mask = std::max(1, std::atoi(e)) - 1;
            // one 8-row block per cluster pair and round: when the last round would leave more than
            // half the pairs idle, its row blocks run as two k1 segments each (a half round;
            // c4: 256 blocks on 74 pairs = 3 rounds + 34 blocks -> 68 half units).  MNB_P2FA_SEG=2
            // splits every row block, MNB_P2FA_SEG=1 none.
            {
                const int64_t pairs = ctx.num_sms / 2, nrb = rs / 8;
                const int64_t full = nrb / pairs * pairs, tail = nrb - full;
                a.full_rb = (tail > 0 && 2 * tail <= pairs) ? full : nrb;  // (full == 0: a short slab, all split)
                if (const char* e = std::getenv("MNB_P2FA_SEG")) a.full_rb = std::atoi(e) == 2 ? 0 : nrb;
            }
            a.halo_seg = op.p2fa_halo.as<int32_t>() + 2048;
            a.rec_t = op.p2fa_rec.as<double2>();
            a.idx_t = op.p2fa_idx.as<int32_t>();
            a.z_t = FP.p2fa_z.as<double2>();
            a.out = x2;
            a.rows = rs;
            a.ldc = (rs + 7) & ~int64_t(7);
            double2* carries = static_cast<double2*>(ctx.ws_carry.ensure(size_t(2 * 1024) * size_t(a.ldc) * 16));
            a.carries = carries;
            launch_p2fa_carries(a, carries, ctx.stream);
            launch_p2fa(a, ctx.num_sms, ctx.stream);
            ctx.launches += 1;
            ctx.launches += 1;
            t.stop();
        } else {  // P2: Pi, Theta, then D (src/srft.cpp:56-57,128)
            EventTimer t(ctx, kernel_ms ? &kernel_ms[1] : nullptr, 1);
            if (chained) {
                HChainArgs a;
                a.in = x1;
                a.ld_in = Ms;
                a.gather = op.at<int32_t>(h.off_perm);
                a.params = op.chain_rec[1].as<double2>();
                a.has_zout = 1;
                a.zout0 = h.at<double2>(h.off_d)[0];
                a.halo = op.at<int32_t>(h.off_halo);  // forward chain of Theta
                a.out = x2;
                a.ld_out = Ms;
                if (blocked) {
                    a.blk_n1 = FP.n1;
                    a.blk_n2 = FP.n2;
                }
                a.rows = rs;
                a.n = n;
                a.chunk = h.ch.chunk;
                a.nchunks = h.ch.nchunks;
                a.max_span = h.max_span;
                launch_hchain(a, ctx.num_sms, ctx.stream);
            } else {
                HStageArgs a = chain_args(op, false, false);
                a.in = x1;
                a.ld_in = Ms;
                a.gather = op.at<int32_t>(h.off_perm);
                a.out = x2;
                a.ld_out = Ms;
                a.out_diag = op.at<double2>(h.off_d);
                a.rows = rs;
                launch_hstage(a, ctx.stream);
            }
            ctx.launches += 1;
            t.stop();
        }
        // F and S (src/srft.cpp:129-131)
        if (blocked || fused)
            fft_rows_blocked(ctx, n, x2, rs, x1, out, ldo, out_row0 + s0, op.at<int32_t>(h.off_sel),
                             op.fb_n2 == FP.n2 ? op.fb_csr.as<int32_t>() : nullptr,
                             kernel_ms ? &kernel_ms[2] : nullptr, kernel_ms ? &kernel_ms[3] : nullptr, fused);
        else
            fft_rows(ctx, n, x2, Ms, rs, x1, Ms, out, ldo, out_row0 + s0, true, op.at<int32_t>(h.off_sel), false,
                     kernel_ms ? &kernel_ms[2] : nullptr, kernel_ms ? &kernel_ms[3] : nullptr,
                     op.fb_n2 == FP.n2 ? op.fb_csr.as<int32_t>() : nullptr);
        if (op.ndups) {
            launch_copy_dups(out, ldo, out_row0 + s0, rs, op.dups.as<int32_t>(), op.ndups, ctx.stream);
            ctx.launches += 1;
        }
        if (ctx.on_slab) ctx.on_slab(out_row0 + s0, rs);
    }
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(MNB_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

int shard_begin(int64_t n, int world, int rank, int64_t* count) {
    const int64_t base = n / world, extra = n % world;
    *count = base + (rank < extra ? 1 : 0);
    return 0;
}

// The all-to-all of the multi-GPU sketch (north_star item 5), as one table per peer h
// (mnb_redistribute_plan in include/minnorm_b200.h):
//   [send_row0, send_rows, send_offset, recv_col0, recv_cols, recv_offset]
// Rank h owns rows mnb_shard_columns(m, world, h) of A and columns mnb_shard_columns(n, world, h).
// pack: block h = A[send_row0 : +send_rows, this rank's columns], column-major (ld send_rows),
//       at element send_offset of the pack buffer;
// slab: this rank's row block (my_rows x n_global, column-major, ld my_rows); peer h's
//       columns land at element recv_offset = recv_col0 * my_rows.
void redistribute_plan(int64_t m, int64_t n_global, int world, int rank, int64_t* plan) {
    int64_t my_rows = 0, my_cols = 0, b = 0;
    mnb_shard_columns(m, world, rank, &b, &my_rows);
    mnb_shard_columns(n_global, world, rank, &b, &my_cols);
    for (int h = 0; h < world; ++h) {
        int64_t r0, rc, c0, cc;
        mnb_shard_columns(m, world, h, &r0, &rc);
        mnb_shard_columns(n_global, world, h, &c0, &cc);
        int64_t* p = plan + 6 * size_t(h);
        p[0] = r0;
        p[1] = rc;
        p[2] = r0 * my_cols;
        p[3] = c0;
        p[4] = cc;
        p[5] = c0 * my_rows;
    }
}

// Column shards -> this rank's row block in ctx.ws_slab: one pack (2D copies) and one grouped
// ncclSend/ncclRecv exchange.  Runs once per solve; both sketches (S and E) read the slab.
void redistribute_rows(Context& ctx, double* seconds) {
    const int64_t m = ctx.m;
    const size_t esz = ctx.esz();
    std::vector<int64_t> plan(size_t(6 * ctx.world));
    redistribute_plan(m, ctx.n_global, ctx.world, ctx.rank, plan.data());
    const int me = ctx.rank;
    const int64_t mh = plan[size_t(6 * me + 1)];
    cudaEvent_t e0 = ctx.event(10), e1 = ctx.event(11);
    MNB_CUDA(cudaEventRecord(e0, ctx.stream));
    unsigned char* pack = static_cast<unsigned char*>(ctx.ws_pack.ensure(size_t(m) * size_t(ctx.n_local) * esz + 16));
    unsigned char* slab =
        static_cast<unsigned char*>(ctx.ws_slab.ensure(size_t(std::max<int64_t>(mh, 1)) * size_t(ctx.n_global) * esz + 16));
    const unsigned char* A = static_cast<const unsigned char*>(ctx.A);
    for (int h = 0; h < ctx.world; ++h) {
        const int64_t* p = &plan[size_t(6 * h)];
        if (p[1] == 0 || ctx.n_local == 0) continue;
        MNB_CUDA(cudaMemcpy2DAsync(pack + size_t(p[2]) * esz, size_t(p[1]) * esz, A + size_t(p[0]) * esz,
                                   size_t(m) * esz, size_t(p[1]) * esz, size_t(ctx.n_local), cudaMemcpyDeviceToDevice,
                                   ctx.stream));
    }
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int h = 0; h < ctx.world; ++h) {
        const int64_t* p = &plan[size_t(6 * h)];
        unsigned char* send = pack + size_t(p[2]) * esz;
        unsigned char* recv = slab + size_t(p[5]) * esz;
        const size_t send_d = size_t(p[1]) * size_t(ctx.n_local) * esz / 8;
        const size_t recv_d = size_t(mh) * size_t(p[4]) * esz / 8;
        if (h == me) {
            if (send_d)
                MNB_CUDA(cudaMemcpyAsync(recv, send, send_d * 8, cudaMemcpyDeviceToDevice, ctx.stream));
            continue;
        }
        if (send_d) nccl_check(ncclSend(send, send_d, ncclDouble, h, ctx.comm, ctx.stream), "ncclSend");
        if (recv_d) nccl_check(ncclRecv(recv, recv_d, ncclDouble, h, ctx.comm, ctx.stream), "ncclRecv");
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
    MNB_CUDA(cudaEventRecord(e1, ctx.stream));
    ctx.slab_ready = true;
    ctx.slab_rows = mh;
    ctx.slab_row0 = plan[size_t(6 * me)];
    if (seconds) {
        MNB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        MNB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        *seconds += ms * 1e-3;
    }
}

void sketch_matrix(Context& ctx, const SrftDev& op, double2* out, double* kernel_ms, double* redistribute_s) {
    const int64_t m = ctx.m, l = op.host->l;
    const int is_real = ctx.dtype == MNB_F64;
    if (!ctx.distributed()) {
        sketch_block(ctx, op, ctx.A, is_real, m, 0, m, out, l, 0, kernel_ms);
        return;
    }
    if (!ctx.slab_ready) redistribute_rows(ctx, redistribute_s);
    // ---- local sketch of this rank's row block ----
    const int64_t mh = ctx.slab_rows;
    if (mh > 0)
        sketch_block(ctx, op, ctx.ws_slab.p, is_real, mh, 0, mh, out + ctx.slab_row0 * l, l, 0, kernel_ms);
    // ---- allgather the sketch columns (every rank runs the replicated QR) ----
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int h = 0; h < ctx.world; ++h) {
        int64_t r0, rows_h;
        mnb_shard_columns(m, ctx.world, h, &r0, &rows_h);
        if (!rows_h) continue;
        double2* blk = out + r0 * l;
        nccl_check(ncclBroadcast(blk, blk, size_t(rows_h) * size_t(l) * 2, ncclDouble, h, ctx.comm, ctx.stream),
                   "ncclBroadcast");
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
}

void dft_vec_to(Context& ctx, int64_t n, const double2* in, double2* out, bool inverse) {
    double2* tmp = static_cast<double2*>(ctx.vec_full[2].ensure(size_t(n) * 16));
    fft_rows(ctx, n, in, 1, 1, tmp, 1, out, 1, 0, false, nullptr, inverse, nullptr, nullptr);
}

void dft_vec(Context& ctx, int64_t n, double2* x, bool inverse) {
    double2* o = static_cast<double2*>(ctx.vec_full[1].ensure(size_t(n) * 16));
    dft_vec_to(ctx, n, x, o, inverse);
    MNB_CUDA(cudaMemcpyAsync(x, o, size_t(n) * 16, cudaMemcpyDeviceToDevice, ctx.stream));
}

void srft_adjoint_vec(Context& ctx, const SrftDev& op, const double2* v, double2* y) {
    const SrftHost& h = *op.host;
    const int64_t n = h.n;
    double2* w = static_cast<double2*>(ctx.vec_full[0].ensure(size_t(n) * 16));
    double2* wf = static_cast<double2*>(ctx.vec_full[1].ensure(size_t(n) * 16));
    // S^* v  (src/srft.cpp:137-139)
    launch_scatter_add_sample(v, h.l, op.at<int32_t>(h.off_sample), h.sampling == MNB_WITH_REPLACEMENT, w, n,
                              ctx.stream);
    // F^{-1} (src/srft.cpp:140)
    dft_vec_to(ctx, n, w, wf, true);
    {  // conj(D), Theta^*, Pi^*, conj(Z)   (src/srft.cpp:141, :64-66)
        HStageArgs a = vec_chain_args(op, false, true);
        a.in = wf;
        a.ld_in = 1;
        a.in_diag = op.at<double2>(h.off_d);
        a.in_diag_conj = 1;
        a.out = w;
        a.ld_out = 1;
        a.scatter = op.at<int32_t>(h.off_perm);
        a.out_diag = op.at<double2>(h.off_zeta);
        a.out_diag_conj = 1;
        a.rows = 1;
        launch_hstage(a, ctx.stream);
    }
    {  // Theta~^*, Pi~^*, conj(Z~)   (src/srft.cpp:67-69)
        HStageArgs a = vec_chain_args(op, true, true);
        a.in = w;
        a.ld_in = 1;
        a.out = y;
        a.ld_out = 1;
        a.scatter = op.at<int32_t>(h.off_perm_tilde);
        a.out_diag = op.at<double2>(h.off_zeta_tilde);
        a.out_diag_conj = 1;
        a.rows = 1;
        launch_hstage(a, ctx.stream);
    }
    ctx.launches += 5;
}

void srft_apply_vec(Context& ctx, const SrftDev& op, const double2* x, double2* y, bool h_only) {
    const SrftHost& h = *op.host;
    const int64_t n = h.n;
    double2* t1 = static_cast<double2*>(ctx.vec_full[0].ensure(size_t(n) * 16));
    double2* t2 = static_cast<double2*>(ctx.vec_full[1].ensure(size_t(n) * 16));
    {
        HStageArgs a = vec_chain_args(op, true, false);
        a.in = x;
        a.ld_in = 1;
        a.gather = op.at<int32_t>(h.off_perm_tilde);
        a.in_diag = op.at<double2>(h.off_zeta_tilde);
        a.out = t1;
        a.ld_out = 1;
        a.out_diag = op.at<double2>(h.off_zeta);
        a.rows = 1;
        launch_hstage(a, ctx.stream);
    }
    {
        HStageArgs a = vec_chain_args(op, false, false);
        a.in = t1;
        a.ld_in = 1;
        a.gather = op.at<int32_t>(h.off_perm);
        a.out = h_only ? y : t2;
        a.ld_out = 1;
        a.out_diag = h_only ? nullptr : op.at<double2>(h.off_d);
        a.rows = 1;
        launch_hstage(a, ctx.stream);
    }
    ctx.launches += 2;
    if (h_only) return;
    double2* tmp = static_cast<double2*>(ctx.vec_full[2].ensure(size_t(n) * 16));
    fft_rows(ctx, n, t2, 1, 1, tmp, 1, y, h.l, 0, true, op.at<int32_t>(h.off_sel), false, nullptr, nullptr);
    if (op.ndups) launch_copy_dups(y, h.l, 0, 1, op.dups.as<int32_t>(), op.ndups, ctx.stream);
}

}  // namespace mnb
