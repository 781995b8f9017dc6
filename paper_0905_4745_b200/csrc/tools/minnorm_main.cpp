// minnorm_b200 -- the reference's command-line front end (tools/minnorm_main.cpp of
// /root/reference/proj) over the C ABI of libminnorm_b200.so: the same subcommands
// (solve, baseline, oracle, gen, bench, selftest), flags, JSON reports, Matrix Market
// files and exit codes (0 success, 1 selftest / solver-quality failure, 2 parse failure,
// 3 dimension mismatch, 4 configuration error; tools/minnorm_main.cpp:29-35,298-316),
// with every solve on the GPU.  Written against include/minnorm_b200.h only: it is the
// C++ shim INTEGRATION.md describes, exercised as a program.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/minnorm_b200.h"

namespace {

using cplx = std::complex<double>;
enum ExitCode { kOk = 0, kQuality = 1, kParse = 2, kDimension = 3, kConfig = 4 };

// ---- errors: C-ABI status -> the reference's exception taxonomy ----------------------
struct Failure {
    int status;
    std::string what;
};

void check(int status) {
    if (status != MNB_OK) throw Failure{status, mnb_last_error()};
}

int exit_code(int status) {
    switch (status) {
        case MNB_ERR_PARSE: return kParse;
        case MNB_ERR_DIMENSION: return kDimension;
        case MNB_ERR_CONFIG:
        case MNB_ERR_INVALID_ARGUMENT: return kConfig;  // ConfigError / std::invalid_argument
        default: return kQuality;                        // RankDeficiencyError, runtime failures
    }
}

// ---- a minimal JSON object writer (insertion order, like nlohmann::json::dump(2)) ----
struct Json {
    std::vector<std::pair<std::string, std::string>> kv;
    static std::string num(double v) {
        if (!std::isfinite(v)) return "null";
        char b[40];
        std::snprintf(b, sizeof b, "%.17g", v);
        return b;
    }
    static std::string str(const std::string& s) {
        std::string o = "\"";
        for (char c : s) {
            if (c == '"' || c == '\\') o += '\\';
            o += c;
        }
        return o + "\"";
    }
    Json& set(const std::string& k, const std::string& raw) {
        kv.emplace_back(k, raw);
        return *this;
    }
    Json& s(const std::string& k, const std::string& v) { return set(k, str(v)); }
    Json& d(const std::string& k, double v) { return set(k, num(v)); }
    Json& i(const std::string& k, long long v) { return set(k, std::to_string(v)); }
    Json& u(const std::string& k, unsigned long long v) { return set(k, std::to_string(v)); }
    Json& b(const std::string& k, bool v) { return set(k, v ? "true" : "false"); }
    std::string dump() const {
        std::string o = "{\n";
        for (size_t k = 0; k < kv.size(); ++k) o += "  " + str(kv[k].first) + ": " + kv[k].second + (k + 1 < kv.size() ? ",\n" : "\n");
        return o + "}";
    }
};

// ---- arguments -------------------------------------------------------------------------
struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    std::map<std::string, bool> flag;
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& flags) {
    Args a;
    for (int k = first; k < argc; ++k) {
        std::string t = argv[k];
        if (t.rfind("--", 0) == 0) {
            const auto eq = t.find('=');
            std::string key = t.substr(2, eq == std::string::npos ? std::string::npos : eq - 2);
            if (std::find(flags.begin(), flags.end(), key) != flags.end()) {
                a.flag[key] = true;
                continue;
            }
            if (eq != std::string::npos) a.opt[key] = t.substr(eq + 1);
            else if (k + 1 < argc) a.opt[key] = argv[++k];
            else throw Failure{MNB_ERR_CONFIG, "option --" + key + " needs a value"};
        } else {
            a.pos.push_back(t);
        }
    }
    return a;
}

double to_double(const std::string& s, const char* what) {
    char* e = nullptr;
    const double v = std::strtod(s.c_str(), &e);
    if (s.empty() || *e) throw Failure{MNB_ERR_CONFIG, std::string(what) + ": not a number: '" + s + "'"};
    return v;
}
unsigned long long to_u64(const std::string& s, const char* what) {
    char* e = nullptr;
    const unsigned long long v = std::strtoull(s.c_str(), &e, 10);
    if (s.empty() || *e || s[0] == '-') throw Failure{MNB_ERR_CONFIG, std::string(what) + ": not an unsigned integer: '" + s + "'"};
    return v;
}

// --seed beats MINNORM_SEED beats 42 (tools/minnorm_main.cpp:45-57)
uint64_t resolve_seed(const Args& a) {
    if (a.opt.count("seed")) return to_u64(a.opt.at("seed"), "--seed");
    if (const char* env = std::getenv("MINNORM_SEED")) {
        char* e = nullptr;
        const unsigned long long v = std::strtoull(env, &e, 10);
        if (!*env || *e) throw Failure{MNB_ERR_CONFIG, std::string("MINNORM_SEED is not an unsigned integer: ") + env};
        return v;
    }
    return 42;
}

int resolve_sampling(const std::string& name) {
    if (name == "without") return MNB_WITHOUT_REPLACEMENT;
    if (name == "with") return MNB_WITH_REPLACEMENT;
    throw Failure{MNB_ERR_CONFIG, "--sampling must be 'with' or 'without', got '" + name + "'"};
}

// ---- problem files ------------------------------------------------------------------------
struct Matrix {
    int64_t rows = 0, cols = 0;
    std::vector<cplx> v;
};

Matrix read_mm(const std::string& path) {
    Matrix M;
    check(mnb_mm_read_dims(path.c_str(), &M.rows, &M.cols));
    M.v.resize(size_t(M.rows * M.cols));
    check(mnb_mm_read(path.c_str(), M.v.data(), M.rows, M.cols));
    return M;
}

std::vector<cplx> read_vec(const std::string& path) {
    Matrix M = read_mm(path);
    if (M.cols != 1)
        throw Failure{MNB_ERR_DIMENSION, "'" + path + "' holds a " + std::to_string(M.rows) + "x" +
                                             std::to_string(M.cols) + " matrix where a vector was expected"};
    return M.v;
}

void write_vec(const std::string& path, const std::vector<cplx>& x) { check(mnb_mm_write(path.c_str(), x.data(), int64_t(x.size()), 1)); }

struct Instance {
    Matrix A;
    std::vector<cplx> b;
};

// ProblemInstance::validate (src/solver.cpp:37-48)
Instance load_instance(const Args& a) {
    if (a.pos.size() < 2) throw Failure{MNB_ERR_CONFIG, "expected the matrix and rhs files"};
    Instance I{read_mm(a.pos[0]), read_vec(a.pos[1])};
    const int64_t m = I.A.rows, n = I.A.cols;
    if (m < 1 || m >= n)
        throw Failure{MNB_ERR_DIMENSION, "problem must be underdetermined: 1 <= m < n, got m=" + std::to_string(m) +
                                             ", n=" + std::to_string(n)};
    if (int64_t(I.b.size()) != m)
        throw Failure{MNB_ERR_DIMENSION, "right-hand side length " + std::to_string(I.b.size()) + " does not match m=" +
                                             std::to_string(m)};
    for (const cplx& z : I.A.v)
        if (!std::isfinite(z.real()) || !std::isfinite(z.imag()))
            throw Failure{MNB_ERR_DIMENSION, "matrix and right-hand side entries must be finite"};
    for (const cplx& z : I.b)
        if (!std::isfinite(z.real()) || !std::isfinite(z.imag()))
            throw Failure{MNB_ERR_DIMENSION, "matrix and right-hand side entries must be finite"};
    return I;
}

double residual(const Matrix& A, const std::vector<cplx>& x, const std::vector<cplx>& b) {
    std::vector<cplx> r(b.size(), 0.0);
    for (int64_t j = 0; j < A.cols; ++j)
        for (int64_t i = 0; i < A.rows; ++i) r[size_t(i)] += A.v[size_t(j * A.rows + i)] * x[size_t(j)];
    double s = 0.0;
    for (size_t i = 0; i < b.size(); ++i) s += std::norm(r[i] - b[i]);
    return std::sqrt(s);
}

double norm(const std::vector<cplx>& x) {
    double s = 0.0;
    for (const cplx& z : x) s += std::norm(z);
    return std::sqrt(s);
}

struct Gpu {
    mnb_context* ctx = nullptr;
    Gpu() {
        int dev = 0;
        if (const char* e = std::getenv("MINNORM_DEVICE")) dev = std::atoi(e);
        check(mnb_context_create(dev, &ctx));
    }
    ~Gpu() { mnb_context_destroy(ctx); }
    void set(const Matrix& A) { check(mnb_set_matrix(ctx, MNB_C128, A.rows, A.cols, 0, A.cols, A.v.data(), A.rows, MNB_HOST)); }
};

Json base_report(const Instance& I) {
    Json j;
    j.s("tool", "minnorm").i("m", I.A.rows).i("n", I.A.cols).s("kernels", std::string("b200:") + mnb_version());
    return j;
}

// ---- subcommands ----------------------------------------------------------------------------
int cmd_solve(const Args& a) {
    const Instance I = load_instance(a);
    mnb_solver_config cfg;
    mnb_solver_config_default(&cfg);
    if (a.opt.count("l")) cfg.sketch_size = int64_t(to_u64(a.opt.at("l"), "--l"));
    if (a.opt.count("alpha")) cfg.alpha = to_double(a.opt.at("alpha"), "--alpha");
    if (a.opt.count("epsilon")) cfg.epsilon = to_double(a.opt.at("epsilon"), "--epsilon");
    cfg.seed = resolve_seed(a);
    const std::string sampling = a.opt.count("sampling") ? a.opt.at("sampling") : "without";
    cfg.sampling = resolve_sampling(sampling);
    if (a.opt.count("max-lsq-iterations")) cfg.lsq_max_iterations = int64_t(to_u64(a.opt.at("max-lsq-iterations"), "--max-lsq-iterations"));
    const std::string out = a.opt.count("out") ? a.opt.at("out") : "x.mtx";
    Gpu g;
    g.set(I.A);
    std::vector<cplx> x(size_t(I.A.cols));
    mnb_solve_report rep;
    check(mnb_solve_randomized(g.ctx, I.b.data(), MNB_HOST, &cfg, x.data(), MNB_HOST, nullptr, &rep));
    write_vec(out, x);
    Json j = base_report(I);
    std::string steps = "[";
    for (int k = 0; k < 5; ++k) steps += Json::num(rep.step_seconds[k]) + (k < 4 ? ", " : "]");
    j.s("subcommand", "solve").i("l", rep.sketch_size).d("alpha", cfg.alpha).d("epsilon", cfg.epsilon).u("seed", cfg.seed)
        .s("sampling", sampling).d("lsq_tau", rep.lsq_tau).i("lsq_iterations", rep.lsq_iterations)
        .b("lsq_converged", rep.lsq_converged).d("residual_norm", rep.residual_norm).d("c_norm_ratio", rep.c_norm_ratio)
        .set("step_times_sec", steps).s("out", out);
    std::printf("%s\n", j.dump().c_str());
    return rep.lsq_converged ? kOk : kQuality;
}

int cmd_baseline(const Args& a) {
    const Instance I = load_instance(a);
    const std::string out = a.opt.count("out") ? a.opt.at("out") : "x.mtx";
    Gpu g;
    g.set(I.A);
    std::vector<cplx> x(size_t(I.A.cols));
    mnb_classical_report rep;
    check(mnb_solve_classical(g.ctx, I.b.data(), MNB_HOST, x.data(), MNB_HOST, &rep));
    write_vec(out, x);
    Json j = base_report(I);
    j.s("subcommand", "baseline").d("residual_norm", residual(I.A, x, I.b)).s("out", out);
    std::printf("%s\n", j.dump().c_str());
    return kOk;
}

int cmd_oracle(const Args& a) {
    const Instance I = load_instance(a);
    Json j = base_report(I);
    j.s("subcommand", "oracle");
    if (a.flag.count("residual")) {
        if (!a.opt.count("solution")) throw Failure{MNB_ERR_CONFIG, "oracle --residual needs --solution <file>"};
        const std::vector<cplx> x = read_vec(a.opt.at("solution"));
        if (int64_t(x.size()) != I.A.cols) throw Failure{MNB_ERR_DIMENSION, "solution length does not match n"};
        const double res = residual(I.A, x, I.b), bn = norm(I.b);
        j.s("solution", a.opt.at("solution")).d("residual_norm", res).d("relative_residual", bn > 0 ? res / bn : 0.0);
        std::printf("%s\n", j.dump().c_str());
        return kOk;
    }
    // the reference's desk-scale reference solve (solve_svd, src/solver.cpp:148-156: m <= 64, n <= 1024);
    // here the exact minimal-norm p of the classical solver on the GPU (same p up to rounding)
    if (I.A.rows > 64 || I.A.cols > 1024)
        throw Failure{MNB_ERR_INVALID_ARGUMENT, "solve_svd: desk-scale reference only (m <= 64, n <= 1024)"};
    const std::string out = a.opt.count("out") ? a.opt.at("out") : "x.mtx";
    Gpu g;
    g.set(I.A);
    std::vector<cplx> p(size_t(I.A.cols));
    mnb_classical_report rep;
    check(mnb_solve_classical(g.ctx, I.b.data(), MNB_HOST, p.data(), MNB_HOST, &rep));
    write_vec(out, p);
    j.d("residual_norm", residual(I.A, p, I.b)).s("out", out);
    std::printf("%s\n", j.dump().c_str());
    return kOk;
}

struct Gen {
    Matrix A;
    std::vector<cplx> b, p;
};

Gen generate(int64_t m, int64_t n, double kappa, uint64_t seed) {
    Gen g;
    g.A.rows = m;
    g.A.cols = n;
    const bool ok = m >= 2 && m < n && kappa >= 1.0;  // else the library reports the DimensionError
    g.A.v.resize(ok ? size_t(m * n) : 1);
    g.b.resize(ok ? size_t(m) : 1);
    g.p.resize(ok ? size_t(n) : 1);
    check(mnb_generate_instance(m, n, kappa, seed, g.A.v.data(), g.b.data(), g.p.data()));
    return g;
}

int cmd_gen(const Args& a) {
    if (!a.opt.count("m") || !a.opt.count("n")) throw Failure{MNB_ERR_CONFIG, "gen needs --m and --n"};
    const int64_t m = int64_t(to_u64(a.opt.at("m"), "--m")), n = int64_t(to_u64(a.opt.at("n"), "--n"));
    const double kappa = a.opt.count("kappa") ? to_double(a.opt.at("kappa"), "--kappa") : 1e6;
    const uint64_t s = resolve_seed(a);
    const std::string prefix = a.opt.count("out") ? a.opt.at("out") : "instance";
    Gen g = generate(m, n, kappa, s);
    check(mnb_mm_write((prefix + "_A.mtx").c_str(), g.A.v.data(), m, n));
    write_vec(prefix + "_b.mtx", g.b);
    write_vec(prefix + "_p.mtx", g.p);
    Json j;
    j.s("tool", "minnorm").s("subcommand", "gen").i("m", m).i("n", n).d("kappa", kappa).u("seed", s)
        .set("files", "[" + Json::str(prefix + "_A.mtx") + ", " + Json::str(prefix + "_b.mtx") + ", " +
                          Json::str(prefix + "_p.mtx") + "]");
    std::printf("%s\n", j.dump().c_str());
    return kOk;
}

uint64_t derive_seed(uint64_t seed, uint64_t tag) {  // RandomStream::derive_seed (src/rng.cpp:37-39)
    auto mix = [](uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    const uint64_t g = 0x9E3779B97F4A7C15ull;
    return mix(mix(seed + g) ^ mix(tag + 2 * g));
}

double seconds_of(const std::function<void()>& fn) {
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double normalized_error(const std::vector<cplx>& x, const std::vector<cplx>& p, double kappa) {  // src/bench.cpp:76-80
    double d = 0.0;
    for (size_t i = 0; i < x.size(); ++i) d += std::norm(x[i] - p[i]);
    return std::sqrt(d) / (kappa * norm(p));
}

// run_benchmark + write_csv (src/bench.cpp:86-141): t0 classical, tr mean of the randomized trials
int cmd_bench(const Args& a) {
    const std::string spec = a.opt.count("grid") ? a.opt.at("grid") : "128:16384:512,256:16384:1024,512:16384:2048";
    const uint64_t trials = a.opt.count("trials") ? to_u64(a.opt.at("trials"), "--trials") : 10;
    const double kappa = a.opt.count("kappa") ? to_double(a.opt.at("kappa"), "--kappa") : 1e6;
    const uint64_t base = resolve_seed(a);
    struct Row {
        unsigned long long m, n, l;
    };
    std::vector<Row> grid;
    std::stringstream ss(spec);
    for (std::string item; std::getline(ss, item, ',');) {
        Row r{};
        if (std::sscanf(item.c_str(), "%llu:%llu:%llu", &r.m, &r.n, &r.l) != 3)
            throw Failure{MNB_ERR_CONFIG, "--grid entries must look like m:n:l, got '" + item + "'"};
        grid.push_back(r);
    }
    if (grid.empty()) throw Failure{MNB_ERR_CONFIG, "--grid is empty"};
    Gpu g;
    std::printf("m,n,l,t0,tr,ratio,eps0,epsr\n");
    bool failed = false;
    for (size_t idx = 0; idx < grid.size(); ++idx) {
        const Row& r = grid[idx];
        try {
            if (!(r.m < r.l && r.l < r.n)) throw Failure{MNB_ERR_CONFIG, "grid row needs m < l < n"};
            if (trials < 1) throw Failure{MNB_ERR_CONFIG, "trials must be at least 1"};
            const Gen gen = generate(int64_t(r.m), int64_t(r.n), kappa, derive_seed(base, 100 + idx));
            g.set(gen.A);
            std::vector<cplx> x0(r.n), x(r.n);
            mnb_classical_report crep;
            const double t0 = seconds_of([&] { check(mnb_solve_classical(g.ctx, gen.b.data(), MNB_HOST, x0.data(), MNB_HOST, &crep)); });
            const double eps0 = normalized_error(x0, gen.p, kappa);
            mnb_solver_config cfg;
            mnb_solver_config_default(&cfg);
            cfg.sketch_size = int64_t(r.l);
            cfg.alpha = 4.0;
            cfg.epsilon = 1e-14 * kappa * std::sqrt(cfg.alpha * double(r.m) / double(r.l));  // bench_epsilon
            double total = 0.0, epsr = 0.0;
            for (uint64_t t = 0; t < trials; ++t) {
                cfg.seed = derive_seed(base, 1000 * (idx + 1) + t);
                mnb_solve_report rep;
                total += seconds_of([&] { check(mnb_solve_randomized(g.ctx, gen.b.data(), MNB_HOST, &cfg, x.data(), MNB_HOST, nullptr, &rep)); });
                epsr = std::max(epsr, normalized_error(x, gen.p, kappa));
            }
            const double tr = total / double(trials);
            std::printf("%llu,%llu,%llu,%.4e,%.4e,%.3f,%.3e,%.3e\n", r.m, r.n, r.l, t0, tr, tr > 0 ? t0 / tr : 0.0, eps0, epsr);
        } catch (const Failure& f) {
            failed = true;
            std::fprintf(stderr, "bench row m=%llu,n=%llu,l=%llu failed: %s\n", r.m, r.n, r.l, f.what.c_str());
        }
    }
    return failed ? kConfig : kOk;
}

// ---- selftest: desk-scale invariant suites through the GPU path (src/selftest.cpp) --------
struct Suite {
    std::string name;
    std::vector<std::pair<std::string, std::function<std::optional<std::string>()>>> checks;
};

struct Rng {  // a plain splitmix64 stream for test vectors (the suites' random inputs)
    uint64_t s;
    double u() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return double((z ^ (z >> 31)) >> 11) * 0x1.0p-53 - 0.5;
    }
    std::vector<cplx> vec(size_t n) {
        std::vector<cplx> v(n);
        for (auto& z : v) z = cplx(u(), u());
        return v;
    }
};

std::string fmt(double v) {
    char b[32];
    std::snprintf(b, sizeof b, "%.3e", v);
    return b;
}

int cmd_selftest(const Args& a) {
    const uint64_t seed = resolve_seed(a);
    const bool corrupt_dft = a.flag.count("corrupt-dft") > 0;  // fault-injection hook (src/selftest.cpp:239)
    Gpu g;
    std::vector<Suite> suites;
    suites.push_back({"rng", {
        {"operator draws match the reference stream (KAT)", [&]() -> std::optional<std::string> {
             mnb_srft* op = nullptr;
             check(mnb_srft_build(8192, int64_t(1) << 20, derive_seed(42, 11), MNB_WITHOUT_REPLACEMENT, &op));
             std::vector<int64_t> s(8192);
             check(mnb_srft_get_field(op, MNB_FIELD_SAMPLE, s.data()));
             mnb_srft_destroy(op);
             const int64_t want[4] = {413293, 426576, 565453, 361359};  // SURVEY 8(c), seed 42, tag 11
             for (int k = 0; k < 4; ++k)
                 if (s[size_t(k)] != want[k]) return "sample[" + std::to_string(k) + "] = " + std::to_string(s[size_t(k)]);
             return std::nullopt;
         }},
    }});
    suites.push_back({"srft", {
        {"dft matches the direct formula", [&]() -> std::optional<std::string> {
             Rng r{seed};
             for (int64_t n = 1; n <= 40; ++n) {
                 std::vector<cplx> x = r.vec(size_t(n)), fast = x;
                 check(mnb_dft(g.ctx, n, fast.data(), 0));
                 if (corrupt_dft) fast[0] += cplx(1e-6, 0.0);
                 double dev = 0.0;
                 for (int64_t k = 0; k < n; ++k) {
                     cplx s = 0.0;
                     for (int64_t j = 0; j < n; ++j) s += x[size_t(j)] * std::polar(1.0, -2.0 * M_PI * double(j * k % n) / double(n));
                     dev += std::norm(fast[size_t(k)] - s / std::sqrt(double(n)));
                 }
                 if (std::sqrt(dev) > 1e-13 * std::max(1.0, norm(x))) return "deviation " + fmt(std::sqrt(dev)) + " at n=" + std::to_string(n);
                 if (std::abs(norm(fast) - norm(x)) > 1e-12 * norm(x)) return "isometry drift at n=" + std::to_string(n);
             }
             return std::nullopt;
         }},
        {"adjoint consistency", [&]() -> std::optional<std::string> {
             Rng r{seed + 1};
             for (int64_t n : {5, 16, 37, 128})
                 for (int mode : {MNB_WITHOUT_REPLACEMENT, MNB_WITH_REPLACEMENT}) {
                     const int64_t l = n / 2 + 1;
                     mnb_srft* op = nullptr;
                     check(mnb_srft_build(l, n, derive_seed(seed, uint64_t(n + mode)), mode, &op));
                     std::vector<cplx> x = r.vec(size_t(n)), v = r.vec(size_t(l)), Tx(static_cast<size_t>(l)), Thv(static_cast<size_t>(n));
                     check(mnb_srft_apply(g.ctx, op, x.data(), Tx.data()));
                     check(mnb_srft_apply_adjoint(g.ctx, op, v.data(), Thv.data()));
                     mnb_srft_destroy(op);
                     cplx lhs = 0.0, rhs = 0.0;
                     for (int64_t k = 0; k < l; ++k) lhs += std::conj(Tx[size_t(k)]) * v[size_t(k)];
                     for (int64_t k = 0; k < n; ++k) rhs += std::conj(x[size_t(k)]) * Thv[size_t(k)];
                     if (std::abs(lhs - rhs) > 1e-12 * norm(x) * norm(v)) return "pairing mismatch " + fmt(std::abs(lhs - rhs));
                 }
             return std::nullopt;
         }},
        {"H unitarity", [&]() -> std::optional<std::string> {
             Rng r{seed + 2};
             for (int64_t n : {2, 3, 17, 64, 1000}) {
                 mnb_srft* op = nullptr;
                 check(mnb_srft_build(std::max<int64_t>(1, n / 2), n, derive_seed(seed, uint64_t(n)), MNB_WITHOUT_REPLACEMENT, &op));
                 std::vector<cplx> x = r.vec(size_t(n)), y(static_cast<size_t>(n));
                 check(mnb_srft_apply_h(g.ctx, op, x.data(), y.data()));
                 mnb_srft_destroy(op);
                 if (std::abs(norm(y) - norm(x)) > 1e-12 * norm(x)) return "norm drift at n=" + std::to_string(n);
             }
             return std::nullopt;
         }},
    }});
    suites.push_back({"minnorm", {
        {"accuracy vs the exact solution", [&]() -> std::optional<std::string> {
             for (uint64_t trial = 0; trial < 5; ++trial) {
                 const Gen gen = generate(8, 512, 1e3, derive_seed(seed, 300 + trial));
                 g.set(gen.A);
                 mnb_solver_config cfg;
                 mnb_solver_config_default(&cfg);
                 cfg.epsilon = 1e-10;
                 cfg.seed = derive_seed(seed, 400 + trial);
                 std::vector<cplx> x(512);
                 mnb_solve_report rep;
                 check(mnb_solve_randomized(g.ctx, gen.b.data(), MNB_HOST, &cfg, x.data(), MNB_HOST, nullptr, &rep));
                 const double e = normalized_error(x, gen.p, 1.0);
                 if (e > 1e-8) return "missed target at trial " + std::to_string(trial) + " (" + fmt(e) + ")";
             }
             return std::nullopt;
         }},
        {"seed determinism (bitwise)", [&]() -> std::optional<std::string> {
             const Gen gen = generate(6, 256, 1e2, derive_seed(seed, 500));
             g.set(gen.A);
             mnb_solver_config cfg;
             mnb_solver_config_default(&cfg);
             std::vector<cplx> x1(256), x2(256);
             mnb_solve_report rep;
             check(mnb_solve_randomized(g.ctx, gen.b.data(), MNB_HOST, &cfg, x1.data(), MNB_HOST, nullptr, &rep));
             check(mnb_solve_randomized(g.ctx, gen.b.data(), MNB_HOST, &cfg, x2.data(), MNB_HOST, nullptr, &rep));
             if (std::memcmp(x1.data(), x2.data(), x1.size() * sizeof(cplx)) != 0) return "two identical runs differ";
             return std::nullopt;
         }},
    }});
    size_t passed = 0, total = 0;
    for (const Suite& s : suites) {
        size_t p = 0;
        for (const auto& [name, fn] : s.checks) {
            std::optional<std::string> failure;
            try {
                failure = fn();
            } catch (const Failure& f) {
                failure = "error: " + f.what;
            }
            if (failure) std::printf("  FAIL %s / %s: %s\n", s.name.c_str(), name.c_str(), failure->c_str());
            else ++p;
        }
        std::printf("suite %s: %zu/%zu passed\n", s.name.c_str(), p, s.checks.size());
        passed += p;
        total += s.checks.size();
    }
    std::printf("selftest: %zu/%zu %s\n", passed, total, passed == total ? "passed" : "passed - FAILURES above");
    return passed == total ? kOk : kQuality;
}

void usage() {
    std::fprintf(stderr,
                 "minnorm_b200 -- randomized minimal-norm solver for underdetermined complex systems (B200)\n"
                 "  solve MATRIX RHS [--l N] [--alpha A] [--epsilon E] [--seed S] [--sampling with|without]\n"
                 "                   [--max-lsq-iterations K] [--out x.mtx]\n"
                 "  baseline MATRIX RHS [--out x.mtx]\n"
                 "  oracle MATRIX RHS [--residual --solution X] [--out x.mtx]\n"
                 "  gen --m M --n N [--kappa K] [--seed S] [--out PREFIX]\n"
                 "  bench [--grid m:n:l,...] [--trials T] [--kappa K] [--seed S]\n"
                 "  selftest [--seed S]\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        usage();
        return argc < 2 ? kConfig : kOk;
    }
    const std::string sub = argv[1];
    try {
        const std::map<std::string, std::vector<std::string>> allowed = {
            {"solve", {"l", "alpha", "epsilon", "seed", "sampling", "max-lsq-iterations", "out"}},
            {"baseline", {"out"}},
            {"oracle", {"residual", "solution", "out"}},
            {"gen", {"m", "n", "kappa", "seed", "out"}},
            {"bench", {"grid", "trials", "kappa", "seed"}},
            {"selftest", {"seed", "corrupt-dft"}}};
        const auto it = allowed.find(sub);
        if (it == allowed.end()) {
            usage();
            return kConfig;
        }
        const Args a = parse_args(argc, argv, 2, {"residual", "corrupt-dft"});
        for (const auto& kv : a.opt)  // CLI11 rejects unknown options (exit 4)
            if (std::find(it->second.begin(), it->second.end(), kv.first) == it->second.end())
                throw Failure{MNB_ERR_CONFIG, "unknown option --" + kv.first + " for '" + sub + "'"};
        const size_t npos_expected = (sub == "solve" || sub == "baseline" || sub == "oracle") ? 2 : 0;
        if (a.pos.size() != npos_expected)
            throw Failure{MNB_ERR_CONFIG, "'" + sub + "' takes " + std::to_string(npos_expected) + " positional arguments"};
        if (sub == "solve") return cmd_solve(a);
        if (sub == "baseline") return cmd_baseline(a);
        if (sub == "oracle") return cmd_oracle(a);
        if (sub == "gen") return cmd_gen(a);
        if (sub == "bench") return cmd_bench(a);
        if (sub == "selftest") return cmd_selftest(a);
        usage();
        return kConfig;
    } catch (const Failure& f) {
        std::fprintf(stderr, "error: %s\n", f.what.c_str());
        return exit_code(f.status);
    }
}
