// Host parameter generation for the SRFT (bit-identical to the reference's
// seeded draws; see host_srft.hpp).  Compiled by the host C++ compiler with
// -ffp-contract=off so every draw rounds exactly like src/rng.cpp.
#include "host_srft.hpp"
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>
#include <deque>
#include <exception>
#include <future>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>

#include "common_host.hpp"

namespace mnb {

namespace {
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr double kTwoPi = 2.0 * 3.14159265358979323846;  // 2.0 * std::numbers::pi, folded exactly
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
inline uint64_t mix(uint64_t z) {  // splitmix64 finalizer
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// Substream tags of build_srft (src/srft.cpp:13-22).
enum : uint64_t { kD = 1, kSample = 2, kTheta = 3, kThetaTilde = 4, kPerm = 5, kPermTilde = 6,
                  kZeta = 7, kZetaTilde = 8 };
// Scan halo: stop once the carried product of |sin| drops below 2^-70.
constexpr double kHaloThreshold = 0x1.0p-70;
}  // namespace

// Persistent host worker pool.  Spawning a fresh set of threads per operator
// (two per solve) costs thread creation plus 8 MiB stack mmap/munmap each,
// whose TLB shootdowns stalled the thread driving the GPU by milliseconds.
// run(width, fn): up to width-1 pool workers join the calling thread in
// calling fn (fn pulls its own work items and returns when none are left).
class WorkerPool {
public:
    static WorkerPool& get() {
        static WorkerPool pool(int(std::max(1u, std::min(64u, std::thread::hardware_concurrency()))));
        return pool;
    }
    void run(int width, const std::function<void()>& fn) {
        auto job = std::make_shared<Job>();
        job->fn = &fn;
        job->slots = std::max(0, std::min(width - 1, int(workers_.size())));
        if (job->slots > 0) {
            std::lock_guard<std::mutex> g(mu_);
            jobs_.push_back(job);
            cv_.notify_all();
        }
        fn();
        {
            std::unique_lock<std::mutex> g(mu_);
            job->slots = 0;  // closed: no new helpers
            jobs_.erase(std::remove(jobs_.begin(), jobs_.end(), job), jobs_.end());
            done_.wait(g, [&] { return job->active == 0; });
        }
    }
    ~WorkerPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
            cv_.notify_all();
        }
        for (auto& t : workers_) t.join();
    }

private:
    struct Job {
        const std::function<void()>* fn = nullptr;
        int slots = 0, active = 0;
    };
    explicit WorkerPool(int n) {
        for (int i = 0; i < n - 1; ++i) workers_.emplace_back([this] { loop(); });
    }
    void loop() {
        std::unique_lock<std::mutex> g(mu_);
        for (;;) {
            cv_.wait(g, [&] {
                if (stop_) return true;
                for (auto& j : jobs_)
                    if (j->slots > 0) return true;
                return false;
            });
            if (stop_) return;
            std::shared_ptr<Job> job;
            for (auto& j : jobs_)
                if (j->slots > 0) {
                    job = j;
                    break;
                }
            --job->slots;
            ++job->active;
            g.unlock();
            (*job->fn)();
            g.lock();
            if (--job->active == 0) done_.notify_all();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::vector<std::shared_ptr<Job>> jobs_;
    bool stop_ = false;
};

// One persistent thread for host_async (tasks run in submission order).
class BackgroundThread {
public:
    static BackgroundThread& get() {
        static BackgroundThread t;
        return t;
    }
    std::future<void> submit(std::function<void()> fn) {
        std::packaged_task<void()> task(std::move(fn));
        auto fut = task.get_future();
        {
            std::lock_guard<std::mutex> g(mu_);
            q_.push_back(std::move(task));
        }
        cv_.notify_one();
        return fut;
    }
    ~BackgroundThread() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_one();
        th_.join();
    }

private:
    BackgroundThread() : th_([this] { loop(); }) {}
    void loop() {
        std::unique_lock<std::mutex> g(mu_);
        for (;;) {
            cv_.wait(g, [&] { return stop_ || !q_.empty(); });
            if (q_.empty()) return;
            auto task = std::move(q_.front());
            q_.pop_front();
            g.unlock();
            task();
            g.lock();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::packaged_task<void()>> q_;
    bool stop_ = false;
    std::thread th_;
};

std::future<void> host_async(std::function<void()> fn) { return BackgroundThread::get().submit(std::move(fn)); }

RandomStream::RandomStream(uint64_t seed) : seed_(seed) {
    uint64_t sm = seed;
    for (auto& w : s_) { sm += kGolden; w = mix(sm); }
}
uint64_t RandomStream::derive_seed(uint64_t tag) const {
    return mix(mix(seed_ + kGolden) ^ mix(tag + 2 * kGolden));
}
uint64_t RandomStream::next_u64() {
    const uint64_t r = rotl(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return r;
}
double RandomStream::uniform_angle() { return kTwoPi * uniform01(); }
void RandomStream::unit_circle(double* z) {
    const double phi = uniform_angle();
    ::sincos(phi, &z[1], &z[0]);
}
void RandomStream::complex_gaussian(double* z) {
    const double u = 1.0 - uniform01();
    const double r = std::sqrt(-std::log(u));
    const double phi = uniform_angle();
    double s, c;
    ::sincos(phi, &s, &c);
    z[0] = r * c;
    z[1] = r * s;
}

uint64_t RandomStream::uniform_below(uint64_t bound) {
    if (bound == 0) throw Error(MNB_ERR_INVALID_ARGUMENT, "uniform_below: bound must be positive");
    // rng.cpp:79-87: accept r >= (0 - bound) % bound.  That threshold is below
    // bound, so for bound <= 2^32 every r >= 2^32 is accepted without computing it.
    for (;;) {
        const uint64_t r = next_u64();
        if ((bound <= (uint64_t(1) << 32) && r >= (uint64_t(1) << 32)) || r >= (0 - bound) % bound)
            return r % bound;
    }
}
// Fisher-Yates (rng.cpp:89-97) with the draws taken in blocks of 64 (same
// stream order) and the swap targets prefetched: the swaps are applied in the
// reference's order, so the permutation is bit-identical; only the cache
// misses of the random p[j] accesses overlap.
void RandomStream::permutation(int32_t* p, int64_t n) {
    for (int64_t i = 0; i < n; ++i) p[i] = int32_t(i);
    constexpr int kBlock = 64;
    uint32_t js[kBlock];
    for (int64_t i = n; i > 1;) {
        const int cnt = int(std::min<int64_t>(kBlock, i - 1));
        for (int k = 0; k < cnt; ++k) {
            js[k] = uint32_t(uniform_below(uint64_t(i - k)));
            __builtin_prefetch(p + js[k], 1);
        }
        for (int k = 0; k < cnt; ++k) std::swap(p[i - 1 - k], p[js[k]]);
        i -= cnt;
    }
}
void RandomStream::sample_indices(int64_t* out, int64_t l, int64_t n, bool without) {
    if (l < 1 || n < 1) throw Error(MNB_ERR_INVALID_ARGUMENT, "sample_indices: l and n must be positive");
    if (without) {
        if (l > n)
            throw Error(MNB_ERR_INVALID_ARGUMENT, "sample_indices: l > n with without-replacement sampling");
        std::vector<int32_t> pool(static_cast<size_t>(n));
        std::iota(pool.begin(), pool.end(), 0);
        for (int64_t i = 0; i < l; ++i) {
            const int64_t j = i + int64_t(uniform_below(uint64_t(n - i)));
            std::swap(pool[size_t(i)], pool[size_t(j)]);
        }
        for (int64_t i = 0; i < l; ++i) out[i] = pool[size_t(i)];
        return;
    }
    for (int64_t i = 0; i < l; ++i) out[i] = int64_t(uniform_below(uint64_t(n)));
}

ChainChunks chain_chunks(int64_t n) {
    ChainChunks c;
    // at least this many chunks per row (the H stage runs one thread per row and chunk; each chunk
    // also walks a ~70-step halo, so short chunks trade redundant steps for parallelism)
    static const int64_t min_chunks = [] {
        const char* e = std::getenv("MNB_CHAIN_MIN_CHUNKS");
        const long v = e ? std::atol(e) : 0;
        return int64_t(v >= 1 ? v : 256);  // (16 -> 256: c2 3.60 -> 3.38 ms, c3 37.9 -> 37.3, profiles/r02/s4h)
    }();
    int64_t chunk = 1024;
    while (chunk > 64 && n / chunk < min_chunks) chunk >>= 1;
    c.chunk = chunk;
    c.nchunks = (n + chunk - 1) / chunk;
    return c;
}

void SrftHost::layout() {
    ch = chain_chunks(n);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    const size_t nn = size_t(n), ll = size_t(l);
    off_d = take(16 * nn);
    off_zeta = take(16 * nn);
    off_zeta_tilde = take(16 * nn);
    off_cssn = take(16 * nn);
    off_cssn_tilde = take(16 * nn);
    off_perm = take(4 * nn);
    off_perm_tilde = take(4 * nn);
    off_sel = take(4 * nn);
    off_halo = take(4 * 4 * size_t(ch.nchunks));
    off_sample = take(4 * ll);
    device_bytes = off;
    off_theta = take(8 * nn);
    off_theta_tilde = take(8 * nn);
    off_sample64 = take(8 * ll);
    total_bytes = off;
}

// Halo starts: per chunk, where the chunked scan may initialise its carry so
// that the neglected contribution is below kHaloThreshold (the carry of the
// chain recurrence decays by |sin(theta_j)| per step).
static void chain_halos(const double* cssn, int64_t n, const ChainChunks& ch, int32_t* fwd, int32_t* adj) {
    std::atomic<int64_t> next{0};
    const std::function<void()> work = [&] {
        for (int64_t c; (c = next.fetch_add(64)) < ch.nchunks;) {
            const int64_t ce = std::min(ch.nchunks, c + 64);
            for (; c < ce; ++c) {
                const int64_t i0 = c * ch.chunk, i1 = std::min(n, i0 + ch.chunk);
                // forward chain: carry flows from high to low indices
                int64_t t = i1;
                if (i1 >= n) t = n - 1;
                else {
                    double p = 1.0;
                    while (t < n - 1 && p > kHaloThreshold) { p *= std::fabs(cssn[2 * t + 1]); ++t; }
                }
                fwd[c] = int32_t(t);
                // adjoint chain: carry flows from low to high indices
                int64_t s = i0;
                double p = 1.0;
                while (s > 0 && p > kHaloThreshold) { --s; p *= std::fabs(cssn[2 * s + 1]); }
                adj[c] = int32_t(s);
            }
        }
    };
    WorkerPool::get().run(int(std::min<int64_t>(16, 1 + ch.nchunks / 256)), work);
}

void SrftHost::derive_first() {
    const int64_t nc = ch.nchunks;
    int32_t* halo = at<int32_t>(off_halo);
    chain_halos(at<double>(off_cssn_tilde), n, ch, halo + nc, halo + 3 * nc);
    span_first = 0;
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t lo = c > 0 ? c * ch.chunk - 1 : 0;
        span_first = std::max<int64_t>(span_first, halo[nc + c] - lo + 1);
    }
    first_derived = true;
}

void SrftHost::derive() {
    const int64_t nc = ch.nchunks;
    int32_t* halo = at<int32_t>(off_halo);
    if (!first_derived) derive_first();
    chain_halos(at<double>(off_cssn), n, ch, halo, halo + 2 * nc);
    max_span = span_first;
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t lo = c > 0 ? c * ch.chunk - 1 : 0;
        max_span = std::max<int64_t>(max_span, halo[c] - lo + 1);
    }
    // selection map: frequency -> first output slot; duplicates listed.
    int32_t* sel = at<int32_t>(off_sel);
    std::fill(sel, sel + n, -1);
    const int64_t* s64 = at<int64_t>(off_sample64);
    int32_t* s32 = at<int32_t>(off_sample);
    dups.clear();
    for (int64_t j = 0; j < l; ++j) {
        const int64_t f = s64[j];
        s32[j] = int32_t(f);
        if (sel[f] < 0) sel[f] = int32_t(j);
        else { dups.push_back(int32_t(j)); dups.push_back(sel[f]); }
    }
    // max multiplicity (src/lsq.cpp:31-39)
    max_mult = 1;
    if (!dups.empty()) {
        std::vector<int64_t> s(s64, s64 + l);
        std::sort(s.begin(), s.end());
        int64_t run = 1;
        for (size_t i = 1; i < s.size(); ++i) {
            run = (s[i] == s[i - 1]) ? run + 1 : 1;
            max_mult = std::max(max_mult, run);
        }
    }
}


void build_srft_host(SrftHost& op, int64_t l, int64_t n, uint64_t stream_seed, int sampling,
                     const BlobAlloc& alloc, const BlobFree& release, int threads, SrftStage* stage) {
    // src/srft.cpp:97-98
    if (n < 2) throw Error(MNB_ERR_INVALID_ARGUMENT, "build_srft: n must be at least 2");
    if (l < 1 || l > n) throw Error(MNB_ERR_INVALID_ARGUMENT, "build_srft: need 1 <= l <= n");
    if (n >= (int64_t(1) << 31)) throw Error(MNB_ERR_UNSUPPORTED, "build_srft: n must be below 2^31");
    const auto t_build0 = std::chrono::steady_clock::now();
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    op.n = n;
    op.l = l;
    op.sampling = sampling;
    op.layout();
    op.blob = alloc(op.total_bytes);
    op.release = release;
    op.first_derived = false;
    const RandomStream stream(stream_seed);
    const bool without = sampling == MNB_WITHOUT_REPLACEMENT;

    // The eight tagged substreams are drawn concurrently (each stream is
    // sequential, as RandomStream requires); the cos/sin of every unit-circle
    // and rotation angle (unit_circle, rng.cpp:62-65; finalize, srft.cpp:80-93)
    // is split into blocks that any idle worker takes as soon as the drawing
    // thread has passed the block's end, so the libm work runs beside the
    // angle draws and the two serial Fisher-Yates permutations.  Unit-circle
    // draws stash phi in the real slot first.  The groups of the first H stage
    // (perm~, theta~, zeta~, zeta) are drawn and evaluated first (SrftStage).
    double* d = op.at<double>(op.off_d);
    double* zeta = op.at<double>(op.off_zeta);
    double* zeta_t = op.at<double>(op.off_zeta_tilde);
    double* theta = op.at<double>(op.off_theta);
    double* theta_t = op.at<double>(op.off_theta_tilde);
    double* cssn = op.at<double>(op.off_cssn);
    double* cssn_t = op.at<double>(op.off_cssn_tilde);
    // angle stream k: 0 d, 1 zeta, 2 zeta~ (unit circle, in place); 3 theta, 4 theta~ (-> cssn)
    std::atomic<int64_t> prog[5];      // angles of stream k drawn so far
    std::atomic<int64_t> next_blk[5];  // next libm block of stream k
    const int64_t count[5] = {n, n, n, n - 1, n - 1};
    for (int k = 0; k < 5; ++k) {
        prog[k] = 0;
        next_blk[k] = 0;
    }
    auto angles_into = [&](RandomStream s, double* out, int k, int64_t stride) {
        constexpr int64_t kStep = 2048;
        for (int64_t i0 = 0; i0 < count[k]; i0 += kStep) {
            const int64_t e = std::min(count[k], i0 + kStep);
            for (int64_t i = i0; i < e; ++i) out[i * stride] = s.uniform_angle();
            prog[k].store(e, std::memory_order_release);
        }
    };
    // libm blocks: 16 per stream (at most 32K angles each), so small operators spread too
    const int64_t blk = std::max<int64_t>(256, std::min<int64_t>(int64_t(1) << 15, n / 16));
    const int64_t nb = (n + blk - 1) / blk;
    auto sincos_block = [&](int k, int64_t b0) {
        if (k < 3) {
            double* z = k == 0 ? d : k == 1 ? zeta : zeta_t;
            const int64_t e = std::min(n, b0 + blk);
            for (int64_t i = b0; i < e; ++i) {
                const double phi = z[2 * i];
                ::sincos(phi, &z[2 * i + 1], &z[2 * i]);
            }
        } else {
            const double* th = k == 3 ? theta : theta_t;
            double* cs = k == 3 ? cssn : cssn_t;
            const int64_t e = std::min(n - 1, b0 + blk);
            for (int64_t i = b0; i < e; ++i) ::sincos(th[i], &cs[2 * i + 1], &cs[2 * i]);
            if (e == n - 1 && b0 <= n - 1) {
                cs[2 * (n - 1)] = 1.0;
                cs[2 * (n - 1) + 1] = 0.0;
            }
        }
    };
    // the next block of stream k whose angles are all drawn: its index, -1 (not drawn yet) or -2 (none left)
    auto take_block = [&](int k) -> int64_t {
        int64_t b = next_blk[k].load();
        while (b < nb) {
            if (prog[k].load(std::memory_order_acquire) < std::min(count[k], (b + 1) * blk)) return -1;
            if (next_blk[k].compare_exchange_weak(b, b + 1)) return b;
        }
        return -2;
    };
    std::atomic<bool> failed{false};
    std::exception_ptr error;
    std::mutex error_mu;
    static const bool tr_tasks = std::getenv("MNB_TRACE") != nullptr;
    double t_task[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::atomic<double> t_sincos_end{0.0};
    double t_first = 0.0;
    auto since0 = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_build0).count(); };
    // first half: perm~ and every libm block of theta~, zeta~, zeta; whoever finishes the last
    // item derives the Theta~ restart points and signals the stage
    std::atomic<int64_t> first_left{1 + 3 * nb};
    auto first_item_done = [&] {
        if (first_left.fetch_sub(1) != 1) return;
        op.derive_first();
        t_first = since0();
        if (stage) stage->signal(1);
    };
    // draw task t: 0..3 the first H stage's groups, 4..7 the rest
    auto draw_task = [&](int t) {
        switch (t) {
            case 0: {
                RandomStream s = stream.substream(kPermTilde);
                s.permutation(op.at<int32_t>(op.off_perm_tilde), n);
                first_item_done();
            } break;
            case 1: angles_into(stream.substream(kThetaTilde), theta_t, 4, 1); break;
            case 2: angles_into(stream.substream(kZetaTilde), zeta_t, 2, 2); break;
            case 3: angles_into(stream.substream(kZeta), zeta, 1, 2); break;
            case 4: { RandomStream s = stream.substream(kPerm); s.permutation(op.at<int32_t>(op.off_perm), n); } break;
            case 5: angles_into(stream.substream(kTheta), theta, 3, 1); break;
            case 6: angles_into(stream.substream(kD), d, 0, 2); break;
            case 7: {
                RandomStream s = stream.substream(kSample);
                s.sample_indices(op.at<int64_t>(op.off_sample64), l, n, without);
            } break;
        }
        if (tr_tasks) t_task[t] = since0();
    };
    // (Holding all four of the other draws back until the first half's libm blocks are claimed
    // measured slower: 12 workers chasing three angle streams mostly spin beside the drawing
    // threads; first half ready 10.0 vs 7.9 ms at n = 2^20, profiles/r02/ab4.)
    // A staged build holds three of the other draws (theta, d, sample: MNB_STAGED_DEFER=0 lifts it)
    // back until the first half's libm blocks are all claimed, so eleven workers instead of eight
    // evaluate them while five draw; perm, the longest, starts at once (c4 280.7 -> 279.4 ms,
    // profiles/r02/ab6).
    static const bool defer_on = !(std::getenv("MNB_STAGED_DEFER") && std::atoi(std::getenv("MNB_STAGED_DEFER")) == 0);
    const bool defer_rest = stage != nullptr && defer_on;
    auto first_blocks_claimed = [&] {
        return next_blk[4].load() >= nb && next_blk[2].load() >= nb && next_blk[1].load() >= nb;
    };
    std::atomic<int> next_first{0}, next_rest{4};
    auto worker = [&] {
        try {
            for (int t; (t = next_first.fetch_add(1)) < 4;) draw_task(t);
            // (the first half's draw tasks are all claimed: its streams advance on their own threads)
            for (;;) {
                bool did = false, left = false;
                for (int k : {4, 2, 1}) {
                    const int64_t b = take_block(k);
                    if (b >= 0) {
                        sincos_block(k, b * blk);
                        first_item_done();
                        did = true;
                        break;
                    }
                    if (b == -1) left = true;
                }
                if (did) continue;
                for (int t = next_rest.load(); t < 8 && (t == 4 || !defer_rest || first_blocks_claimed());) {
                    if (next_rest.compare_exchange_weak(t, t + 1)) {
                        draw_task(t);
                        did = true;
                        break;
                    }
                }
                if (did) continue;
                if (next_rest.load() >= 8)  // every draw task is claimed: the rest's blocks as they come
                    for (int k : {3, 0}) {
                        const int64_t b = take_block(k);
                        if (b >= 0) {
                            sincos_block(k, b * blk);
                            did = true;
                            break;
                        }
                        if (b == -1) left = true;
                    }
                else
                    left = true;
                if (did) continue;
                if (!left || failed.load()) break;
                std::this_thread::yield();
            }
            if (tr_tasks) {
                const double te = since0();
                double cur = t_sincos_end.load();
                while (te > cur && !t_sincos_end.compare_exchange_weak(cur, te)) {}
            }
        } catch (...) {
            {
                std::lock_guard<std::mutex> g(error_mu);
                if (!error) error = std::current_exception();
            }
            failed = true;
            if (stage) stage->signal(2);
        }
    };
    {
        // one worker per 512 indices up to `threads` (tiny operators are drawn in microseconds)
        const int nt = int(std::max<int64_t>(1, std::min<int64_t>(threads, n / 512)));
        const std::function<void()> work = worker;
        WorkerPool::get().run(nt, work);
    }
    if (error) std::rethrow_exception(error);
    static const bool tr = std::getenv("MNB_TRACE") != nullptr;
    const auto t_drawn = std::chrono::steady_clock::now();
    op.derive();
    if (tr) {
        const double ms_draw = std::chrono::duration<double, std::milli>(t_drawn - t_build0).count();
        const double ms_derive =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_drawn).count();
        std::fprintf(stderr, "[mnb] build_srft n=%lld threads=%d: draw %.2f ms, derive %.2f ms; tasks done at perm~ %.2f "
                             "theta~ %.2f zeta~ %.2f zeta %.2f perm %.2f theta %.2f d %.2f sample %.2f; first half ready "
                             "%.2f, last sincos %.2f ms\n",
                     (long long)n, threads, ms_draw, ms_derive, t_task[0], t_task[1], t_task[2], t_task[3], t_task[4],
                     t_task[5], t_task[6], t_task[7], t_first, t_sincos_end.load());
    }
}

}  // namespace mnb
