// ============================================================================
// oracle/minnorm_oracle.cpp  --  TEST INFRASTRUCTURE ONLY (the CPU checker).
//
// A plain C++ restatement of the reference's randomized min-norm hot path,
// used exclusively by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs.  The shipped product
// (paper_0905_4745_b200/) never links, imports or calls anything here.
//
// Every routine cites the reference file:line it restates
// (paths relative to /root/reference/proj).  The arithmetic follows the
// reference's SCALAR backend expression-for-expression (no FMA contraction:
// build with -ffp-contract=off), so results are bit-identical to the
// reference scalar kernels where the algorithm is the same.
//
// Parity pins:
//   * rng / kernels are checked bit-for-bit against the reference's own
//     src/rng.cpp + src/kernels_scalar.cpp compiled verbatim into
//     oracle/_ref/libminnorm_ref.so (oracle/Makefile, target `ref`);
//   * fft / srft are checked against the reference tests' known answers
//     (tests/test_fft.cpp, tests/test_srft.cpp) and dense oracles
//     (tests/test_support.hpp) restated in tests/.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <thread>
#include <vector>

namespace oracle {

using Complex = std::complex<double>;
static constexpr double kPi = 3.14159265358979323846;  // == std::numbers::pi

// ---------------------------------------------------------------- rng -------
// src/rng.cpp:12-30 (splitmix64 + rotl), :32-52 (ctor, derive_seed, next_u64)
static constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t smix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct Rng {
    uint64_t seed;
    uint64_t s[4];
    explicit Rng(uint64_t sd) : seed(sd) {
        uint64_t sm = sd;
        for (auto& w : s) { sm += kGolden; w = smix(sm); }
    }
    uint64_t derive(uint64_t tag) const {  // rng.cpp:37-39
        return smix(smix(seed + kGolden) ^ smix(tag + 2 * kGolden));
    }
    Rng sub(uint64_t tag) const { return Rng(derive(tag)); }
    uint64_t next() {  // rng.cpp:41-52 (xoshiro256++)
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
        s[2] ^= t; s[3] = rotl(s[3], 45);
        return r;
    }
    double u01() { return double(next() >> 11) * 0x1.0p-53; }       // rng.cpp:54-56
    double angle() { return 2.0 * kPi * u01(); }                      // rng.cpp:58-60
    Complex unit() { const double p = angle(); return {std::cos(p), std::sin(p)}; }  // :62-65
    double sign() { return (next() >> 63) ? 1.0 : -1.0; }             // :67-69
    Complex cgauss() {                                                // :71-77
        const double u = 1.0 - u01();
        const double r = std::sqrt(-std::log(u));
        const double p = angle();
        return {r * std::cos(p), r * std::sin(p)};
    }
    uint64_t below(uint64_t bound) {                                  // :79-87
        if (bound == 0) throw std::invalid_argument("uniform_below: bound must be positive");
        const uint64_t thr = (0 - bound) % bound;
        for (;;) { const uint64_t r = next(); if (r >= thr) return r % bound; }
    }
    std::vector<int64_t> permutation(size_t n) {                      // :89-97
        std::vector<int64_t> p(n);
        std::iota(p.begin(), p.end(), int64_t{0});
        for (size_t i = n; i > 1; --i) {
            const size_t j = size_t(below(i));
            std::swap(p[i - 1], p[j]);
        }
        return p;
    }
    std::vector<int64_t> sample(size_t l, size_t n, bool without) {   // :99-117
        if (l < 1 || n < 1) throw std::invalid_argument("sample_indices: l and n must be positive");
        if (without) {
            if (l > n) throw std::invalid_argument("sample_indices: l > n with without-replacement sampling");
            std::vector<int64_t> pool(n);
            std::iota(pool.begin(), pool.end(), int64_t{0});
            for (size_t i = 0; i < l; ++i) {
                const size_t j = i + size_t(below(n - i));
                std::swap(pool[i], pool[j]);
            }
            pool.resize(l);
            return pool;
        }
        std::vector<int64_t> out(l);
        for (auto& v : out) v = int64_t(below(n));
        return out;
    }
};

// ------------------------------------------------------------- kernels ------
// src/kernels_scalar.cpp:7-13
static void cmul(Complex* y, const Complex* x, const Complex* d, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = x[i] * d[i];
}
static void cmul_conj(Complex* y, const Complex* x, const Complex* d, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = x[i] * std::conj(d[i]);
}
// src/kernels_scalar.cpp:15-33
static void rotation_chain(Complex* x, const double* cs, const double* sn, size_t n, bool adjoint) {
    if (n < 2) return;
    if (!adjoint) {
        for (size_t j = n - 1; j-- > 0;) {
            const Complex a = x[j], b = x[j + 1];
            x[j] = cs[j] * a + sn[j] * b;
            x[j + 1] = -sn[j] * a + cs[j] * b;
        }
    } else {
        for (size_t j = 0; j + 1 < n; ++j) {
            const Complex a = x[j], b = x[j + 1];
            x[j] = cs[j] * a - sn[j] * b;
            x[j + 1] = sn[j] * a + cs[j] * b;
        }
    }
}
// src/kernels_scalar.cpp:35-46
static void fft_stage(Complex* x, const Complex* tw, size_t n, size_t gap, bool conj_tw) {
    for (size_t base = 0; base < n; base += 2 * gap)
        for (size_t j = 0; j < gap; ++j) {
            const Complex w = conj_tw ? std::conj(tw[j]) : tw[j];
            const Complex u = x[base + j];
            const Complex v = x[base + j + gap] * w;
            x[base + j] = u + v;
            x[base + j + gap] = u - v;
        }
}

// ----------------------------------------------------------------- fft ------
// src/fft.cpp:14-131
static bool is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }
static size_t next_pow2(size_t n) { size_t p = 1; while (p < n) p <<= 1; return p; }

struct Fft {
    size_t n;
    bool pow2;
    double scale;
    std::vector<size_t> bitrev;
    std::vector<Complex> stage_tw;
    std::unique_ptr<Fft> padded;
    std::vector<Complex> chirp, chirp_spec;

    explicit Fft(size_t n_) : n(n_), pow2(is_pow2(n_)), scale(n_ ? 1.0 / std::sqrt(double(n_)) : 1.0) {
        if (n == 0) throw std::invalid_argument("Fft: length must be positive");
        if (n == 1) return;
        if (pow2) {  // fft.cpp:38-47
            bitrev.resize(n);
            bitrev[0] = 0;
            for (size_t i = 1; i < n; ++i) bitrev[i] = (bitrev[i >> 1] >> 1) | ((i & 1) ? n >> 1 : 0);
            stage_tw.reserve(n - 1);
            for (size_t gap = 1; gap < n; gap <<= 1)
                for (size_t j = 0; j < gap; ++j)
                    stage_tw.push_back(std::polar(1.0, -kPi * double(j) / double(gap)));
            return;
        }
        // Bluestein, fft.cpp:49-62
        padded = std::make_unique<Fft>(next_pow2(2 * n - 1));
        const size_t np = padded->n;
        chirp.resize(n);
        for (size_t k = 0; k < n; ++k) {
            const size_t t = (k * k) % (2 * n);
            chirp[k] = std::polar(1.0, -kPi * double(t) / double(n));
        }
        std::vector<Complex> b(np, Complex(0.0, 0.0));
        b[0] = std::conj(chirp[0]);
        for (size_t k = 1; k < n; ++k) b[k] = b[np - k] = std::conj(chirp[k]);
        padded->raw_pow2(b.data(), false);
        chirp_spec = std::move(b);
    }
    void raw_pow2(Complex* x, bool conj_tw) const {  // fft.cpp:65-76
        for (size_t i = 0; i < n; ++i) { const size_t j = bitrev[i]; if (i < j) std::swap(x[i], x[j]); }
        const Complex* tw = stage_tw.data();
        for (size_t gap = 1; gap < n; gap <<= 1) { fft_stage(x, tw, n, gap, conj_tw); tw += gap; }
    }
    void raw_bluestein(Complex* x) const {  // fft.cpp:78-88
        const size_t np = padded->n;
        std::vector<Complex> a(np, Complex(0.0, 0.0));
        cmul(a.data(), x, chirp.data(), n);
        padded->raw_pow2(a.data(), false);
        cmul(a.data(), a.data(), chirp_spec.data(), np);
        padded->raw_pow2(a.data(), true);
        const double s = 1.0 / double(np);
        for (size_t i = 0; i < np; ++i) a[i] *= s;
        cmul(x, a.data(), chirp.data(), n);
    }
    void forward(Complex* x) const {  // fft.cpp:90-97
        if (n == 1) return;
        if (pow2) raw_pow2(x, false); else raw_bluestein(x);
        for (size_t i = 0; i < n; ++i) x[i] *= scale;
    }
    void inverse(Complex* x) const {  // fft.cpp:99-110
        if (n == 1) return;
        if (pow2) {
            raw_pow2(x, true);
            for (size_t i = 0; i < n; ++i) x[i] *= scale;
            return;
        }
        for (size_t i = 0; i < n; ++i) x[i] = std::conj(x[i]);
        forward(x);
        for (size_t i = 0; i < n; ++i) x[i] = std::conj(x[i]);
    }
};

static std::shared_ptr<const Fft> fft_plan(size_t n) {  // fft.cpp:112-119
    static std::mutex mu;
    static std::map<size_t, std::shared_ptr<const Fft>> cache;
    std::scoped_lock lock(mu);
    auto& slot = cache[n];
    if (!slot) slot = std::make_shared<Fft>(n);
    return slot;
}

// ---------------------------------------------------------------- srft ------
// include/minnorm/srft.hpp:21-59 ; src/srft.cpp:13-168
struct Srft {
    size_t n = 0, l = 0;
    bool without = true;
    std::vector<Complex> d, zeta, zeta_tilde;
    std::vector<int64_t> sample, perm, perm_tilde;
    std::vector<double> theta, theta_tilde;
    std::vector<double> cos_theta, sin_theta, cos_theta_tilde, sin_theta_tilde;
    std::shared_ptr<const Fft> fft;

    void finalize() {  // srft.cpp:80-93
        const size_t chain = n >= 1 ? n - 1 : 0;
        cos_theta.resize(chain); sin_theta.resize(chain);
        cos_theta_tilde.resize(chain); sin_theta_tilde.resize(chain);
        for (size_t j = 0; j < chain; ++j) {
            cos_theta[j] = std::cos(theta[j]);
            sin_theta[j] = std::sin(theta[j]);
            cos_theta_tilde[j] = std::cos(theta_tilde[j]);
            sin_theta_tilde[j] = std::sin(theta_tilde[j]);
        }
        fft = fft_plan(n);
    }
    static void gather(Complex* scratch, Complex* x, const std::vector<int64_t>& p) {  // srft.cpp:36-40
        const size_t n = p.size();
        for (size_t i = 0; i < n; ++i) scratch[i] = x[p[i]];
        std::copy(scratch, scratch + n, x);
    }
    static void scatter(Complex* scratch, Complex* x, const std::vector<int64_t>& p) {  // :42-46
        const size_t n = p.size();
        for (size_t i = 0; i < n; ++i) scratch[p[i]] = x[i];
        std::copy(scratch, scratch + n, x);
    }
    void apply_h_inplace(Complex* x, Complex* scratch) const {  // srft.cpp:49-58
        cmul(x, x, zeta_tilde.data(), n);
        gather(scratch, x, perm_tilde);
        rotation_chain(x, cos_theta_tilde.data(), sin_theta_tilde.data(), n, false);
        cmul(x, x, zeta.data(), n);
        gather(scratch, x, perm);
        rotation_chain(x, cos_theta.data(), sin_theta.data(), n, false);
    }
    void apply_h_adjoint_inplace(Complex* x, Complex* scratch) const {  // srft.cpp:61-70
        rotation_chain(x, cos_theta.data(), sin_theta.data(), n, true);
        scatter(scratch, x, perm);
        cmul_conj(x, x, zeta.data(), n);
        rotation_chain(x, cos_theta_tilde.data(), sin_theta_tilde.data(), n, true);
        scatter(scratch, x, perm_tilde);
        cmul_conj(x, x, zeta_tilde.data(), n);
    }
    // srft.cpp:123-133 ; w is length-n scratch, out length l
    void apply(const Complex* x, Complex* out, Complex* w, Complex* scratch) const {
        std::copy(x, x + n, w);
        apply_h_inplace(w, scratch);
        cmul(w, w, d.data(), n);
        fft->forward(w);
        for (size_t j = 0; j < l; ++j) out[j] = w[sample[j]];
    }
    // srft.cpp:135-145
    void apply_adjoint(const Complex* v, Complex* out) const {
        std::fill(out, out + n, Complex(0.0, 0.0));
        for (size_t j = 0; j < l; ++j) out[sample[j]] += v[j];
        fft->inverse(out);
        cmul_conj(out, out, d.data(), n);
        std::vector<Complex> scratch(n);
        apply_h_adjoint_inplace(out, scratch.data());
    }
};

// srft.cpp:95-113 (tags srft.cpp:13-22)
static Srft* build_srft(size_t l, size_t n, uint64_t stream_seed, bool without) {
    if (n < 2) throw std::invalid_argument("build_srft: n must be at least 2");
    if (l < 1 || l > n) throw std::invalid_argument("build_srft: need 1 <= l <= n");
    Rng stream(stream_seed);
    auto* op = new Srft;
    op->n = n; op->l = l; op->without = without;
    { Rng s = stream.sub(1); op->d.resize(n); for (auto& v : op->d) v = s.unit(); }
    { Rng s = stream.sub(2); op->sample = s.sample(l, n, without); }
    { Rng s = stream.sub(3); op->theta.resize(n - 1); for (auto& v : op->theta) v = s.angle(); }
    { Rng s = stream.sub(4); op->theta_tilde.resize(n - 1); for (auto& v : op->theta_tilde) v = s.angle(); }
    { Rng s = stream.sub(5); op->perm = s.permutation(n); }
    { Rng s = stream.sub(6); op->perm_tilde = s.permutation(n); }
    { Rng s = stream.sub(7); op->zeta.resize(n); for (auto& v : op->zeta) v = s.unit(); }
    { Rng s = stream.sub(8); op->zeta_tilde.resize(n); for (auto& v : op->zeta_tilde) v = s.unit(); }
    op->finalize();
    return op;
}

}  // namespace oracle

// ============================================================ C exports =====
using oracle::Complex;
using oracle::Rng;
using oracle::Srft;

namespace {
thread_local char g_err[512];
int fail(const std::exception& e) {
    std::snprintf(g_err, sizeof g_err, "%s", e.what());
    return -1;
}
}  // namespace

extern "C" {

const char* or_last_error() { return g_err; }

// ---- rng (src/rng.cpp) ----
uint64_t or_derive_seed(uint64_t seed, uint64_t tag) { return Rng(seed).derive(tag); }
void or_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.next();
}
// kind: 0 u01, 1 angle, 2 unit_circle (2 doubles), 3 sign, 4 complex_gaussian (2 doubles)
void or_rng_draw(uint64_t seed, int kind, int64_t count, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) {
        switch (kind) {
            case 0: out[i] = r.u01(); break;
            case 1: out[i] = r.angle(); break;
            case 2: { Complex z = r.unit(); out[2 * i] = z.real(); out[2 * i + 1] = z.imag(); } break;
            case 3: out[i] = r.sign(); break;
            case 4: { Complex z = r.cgauss(); out[2 * i] = z.real(); out[2 * i + 1] = z.imag(); } break;
        }
    }
}
int or_rng_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out) {
    try { Rng r(seed); for (int64_t i = 0; i < count; ++i) out[i] = r.below(bound); return 0; }
    catch (const std::exception& e) { return fail(e); }
}
int or_rng_permutation(uint64_t seed, int64_t n, int64_t* out) {
    Rng r(seed); auto p = r.permutation(size_t(n)); std::copy(p.begin(), p.end(), out); return 0;
}
int or_rng_sample(uint64_t seed, int64_t l, int64_t n, int without, int64_t* out) {
    try { Rng r(seed); auto p = r.sample(size_t(l), size_t(n), without != 0); std::copy(p.begin(), p.end(), out); return 0; }
    catch (const std::exception& e) { return fail(e); }
}

// ---- kernels (src/kernels_scalar.cpp) ----
void or_cmul(double* y, const double* x, const double* d, int64_t n, int conj) {
    if (conj) oracle::cmul_conj((Complex*)y, (const Complex*)x, (const Complex*)d, size_t(n));
    else oracle::cmul((Complex*)y, (const Complex*)x, (const Complex*)d, size_t(n));
}
void or_rotation_chain(double* x, const double* cs, const double* sn, int64_t n, int adjoint) {
    oracle::rotation_chain((Complex*)x, cs, sn, size_t(n), adjoint != 0);
}
void or_fft_stage(double* x, const double* tw, int64_t n, int64_t gap, int conj_tw) {
    oracle::fft_stage((Complex*)x, (const Complex*)tw, size_t(n), size_t(gap), conj_tw != 0);
}

// ---- fft (src/fft.cpp) ----
int or_fft(double* x, int64_t n, int inverse) {
    try {
        auto p = oracle::fft_plan(size_t(n));
        if (inverse) p->inverse((Complex*)x); else p->forward((Complex*)x);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// ---- srft (src/srft.cpp) ----
void* or_srft_build(int64_t l, int64_t n, uint64_t stream_seed, int without) {
    try { return oracle::build_srft(size_t(l), size_t(n), stream_seed, without != 0); }
    catch (const std::exception& e) { fail(e); return nullptr; }
}
// Operator from caller-supplied fields (trivial operators, hand-built KATs).
void* or_srft_from_fields(int64_t l, int64_t n, int without, const double* d, const int64_t* sample,
                          const double* theta, const double* theta_tilde, const int64_t* perm,
                          const int64_t* perm_tilde, const double* zeta, const double* zeta_tilde) {
    auto* op = new Srft;
    op->n = size_t(n); op->l = size_t(l); op->without = without != 0;
    op->d.assign((const Complex*)d, (const Complex*)d + n);
    op->zeta.assign((const Complex*)zeta, (const Complex*)zeta + n);
    op->zeta_tilde.assign((const Complex*)zeta_tilde, (const Complex*)zeta_tilde + n);
    op->sample.assign(sample, sample + l);
    op->perm.assign(perm, perm + n);
    op->perm_tilde.assign(perm_tilde, perm_tilde + n);
    op->theta.assign(theta, theta + (n - 1));
    op->theta_tilde.assign(theta_tilde, theta_tilde + (n - 1));
    op->finalize();
    return op;
}
void or_srft_free(void* h) { delete static_cast<Srft*>(h); }

// field ids: 0 d,1 zeta,2 zeta_tilde (complex n); 3 theta,4 theta_tilde,5 cos_theta,6 sin_theta,
//            7 cos_theta_tilde,8 sin_theta_tilde (real n-1); 9 perm,10 perm_tilde (int64 n); 11 sample (int64 l)
int or_srft_field(void* h, int field, void* out) {
    const Srft& op = *static_cast<Srft*>(h);
    const size_t n = op.n;
    auto cpyc = [&](const std::vector<Complex>& v) { std::memcpy(out, v.data(), v.size() * sizeof(Complex)); };
    auto cpyd = [&](const std::vector<double>& v) { std::memcpy(out, v.data(), v.size() * sizeof(double)); };
    auto cpyi = [&](const std::vector<int64_t>& v) { std::memcpy(out, v.data(), v.size() * sizeof(int64_t)); };
    switch (field) {
        case 0: cpyc(op.d); break;
        case 1: cpyc(op.zeta); break;
        case 2: cpyc(op.zeta_tilde); break;
        case 3: cpyd(op.theta); break;
        case 4: cpyd(op.theta_tilde); break;
        case 5: cpyd(op.cos_theta); break;
        case 6: cpyd(op.sin_theta); break;
        case 7: cpyd(op.cos_theta_tilde); break;
        case 8: cpyd(op.sin_theta_tilde); break;
        case 9: cpyi(op.perm); break;
        case 10: cpyi(op.perm_tilde); break;
        case 11: cpyi(op.sample); break;
        default: return -1;
    }
    (void)n;
    return 0;
}

void or_srft_apply_h(void* h, const double* x, double* out) {
    const Srft& op = *static_cast<Srft*>(h);
    std::vector<Complex> scratch(op.n);
    std::copy((const Complex*)x, (const Complex*)x + op.n, (Complex*)out);
    op.apply_h_inplace((Complex*)out, scratch.data());
}
void or_srft_apply(void* h, const double* x, double* out) {
    const Srft& op = *static_cast<Srft*>(h);
    std::vector<Complex> w(op.n), scratch(op.n);
    op.apply((const Complex*)x, (Complex*)out, w.data(), scratch.data());
}
void or_srft_apply_adjoint(void* h, const double* v, double* out) {
    static_cast<Srft*>(h)->apply_adjoint((const Complex*)v, (Complex*)out);
}

// The sketch T·B with B = A^H (src/solver.cpp:76,81 ; src/lsq.cpp:56 ; src/srft.cpp:147-153),
// without materialising B: column j of the output is T·conj(A[row0+j, :]).
// A is column-major m×n (complex, or real when is_real) with leading dimension lda.
// out: l×nrows column-major (ld = l).  Column loop parallelised over `threads`
// (permitted by SPEC.md:207; results independent of the thread count).
int or_srft_sketch_rows(void* h, const void* A, int is_real, int64_t lda, int64_t row0, int64_t nrows,
                        double* out, int threads) {
    const Srft& op = *static_cast<Srft*>(h);
    const size_t n = op.n, l = op.l;
    if (threads < 1) threads = 1;
    auto work = [&](int64_t jb, int64_t je) {
        std::vector<Complex> col(n), w(n), scratch(n);
        for (int64_t j = jb; j < je; ++j) {
            const int64_t row = row0 + j;
            if (is_real) {
                const double* Ar = static_cast<const double*>(A);
                for (size_t k = 0; k < n; ++k) col[k] = Complex(Ar[row + int64_t(k) * lda], 0.0);
            } else {
                const Complex* Ac = static_cast<const Complex*>(A);
                for (size_t k = 0; k < n; ++k) col[k] = std::conj(Ac[row + int64_t(k) * lda]);
            }
            op.apply(col.data(), (Complex*)out + size_t(j) * l, w.data(), scratch.data());
        }
    };
    std::vector<std::thread> pool;
    const int64_t per = (nrows + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t b = t * per, e = std::min<int64_t>(nrows, b + per);
        if (b < e) pool.emplace_back(work, b, e);
    }
    for (auto& th : pool) th.join();
    return 0;
}

// B·v = A^H v (n-vector) and B^H r = A r (m-vector) with a threaded column split;
// src/lsq.cpp:71-73 GEMVs.  Deterministic: fixed partition + fixed reduction order.
void or_gemv_AH(const void* A, int is_real, int64_t m, int64_t n, int64_t lda, const double* v, double* out, int threads) {
    const Complex* vv = (const Complex*)v;
    Complex* o = (Complex*)out;
    auto work = [&](int64_t kb, int64_t ke) {
        for (int64_t k = kb; k < ke; ++k) {
            Complex acc(0.0, 0.0);
            if (is_real) {
                const double* col = static_cast<const double*>(A) + k * lda;
                for (int64_t i = 0; i < m; ++i) acc += col[i] * vv[i];
            } else {
                const Complex* col = static_cast<const Complex*>(A) + k * lda;
                for (int64_t i = 0; i < m; ++i) acc += std::conj(col[i]) * vv[i];
            }
            o[k] = acc;
        }
    };
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    const int64_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t b = t * per, e = std::min<int64_t>(n, b + per);
        if (b < e) pool.emplace_back(work, b, e);
    }
    for (auto& th : pool) th.join();
}
void or_gemv_A(const void* A, int is_real, int64_t m, int64_t n, int64_t lda, const double* r, double* out, int threads) {
    const Complex* rr = (const Complex*)r;
    if (threads < 1) threads = 1;
    std::vector<std::vector<Complex>> part(static_cast<size_t>(threads), std::vector<Complex>(static_cast<size_t>(m)));
    auto work = [&](int t, int64_t kb, int64_t ke) {
        auto& acc = part[size_t(t)];
        for (int64_t k = kb; k < ke; ++k) {
            const Complex rk = rr[k];
            if (is_real) {
                const double* col = static_cast<const double*>(A) + k * lda;
                for (int64_t i = 0; i < m; ++i) acc[i] += col[i] * rk;
            } else {
                const Complex* col = static_cast<const Complex*>(A) + k * lda;
                for (int64_t i = 0; i < m; ++i) acc[i] += col[i] * rk;
            }
        }
    };
    std::vector<std::thread> pool;
    const int64_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t b = t * per, e = std::min<int64_t>(n, b + per);
        if (b < e) pool.emplace_back(work, t, b, e);
    }
    for (auto& th : pool) th.join();
    Complex* o = (Complex*)out;
    for (int64_t i = 0; i < m; ++i) {
        Complex s(0.0, 0.0);
        for (int t = 0; t < threads; ++t) s += part[size_t(t)][size_t(i)];
        o[i] = s;
    }
}

}  // extern "C"
