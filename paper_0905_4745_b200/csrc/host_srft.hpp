// Host side of the SRFT operator: the reference's seeded RandomStream
// (bit-identical draws) and a parallel build_srft that writes the parameters
// straight into one upload-ready blob.
#pragma once

#include <cstddef>
#include <cstdint>
#include <condition_variable>
#include <functional>
#include <future>
#include <mutex>
#include <vector>

namespace mnb {

// xoshiro256++ seeded through splitmix64 -- the generator the reference fixes
// in include/minnorm/rng.hpp:8-14 (src/rng.cpp:12-117).  Same API names.
class RandomStream {
public:
    explicit RandomStream(uint64_t seed = 42);
    uint64_t seed() const { return seed_; }
    uint64_t derive_seed(uint64_t tag) const;                        // rng.cpp:37-39
    RandomStream substream(uint64_t tag) const { return RandomStream(derive_seed(tag)); }
    uint64_t next_u64();                                             // rng.cpp:41-52
    double uniform01() { return double(next_u64() >> 11) * 0x1.0p-53; }
    double uniform_angle();                                          // rng.cpp:58-60
    void unit_circle(double* re_im);                                 // rng.cpp:62-65
    double sign() { return (next_u64() >> 63) ? 1.0 : -1.0; }
    void complex_gaussian(double* re_im);                            // rng.cpp:71-77
    uint64_t uniform_below(uint64_t bound);                          // rng.cpp:79-87
    void permutation(int32_t* p, int64_t n);                         // rng.cpp:89-97
    void sample_indices(int64_t* out, int64_t l, int64_t n, bool without);  // rng.cpp:99-117

private:
    uint64_t seed_;
    uint64_t s_[4];
};

// Chunking of the rotation-chain scans (see k_hstage.cu).
struct ChainChunks {
    int64_t chunk = 0;    // columns per chunk
    int64_t nchunks = 0;
};
ChainChunks chain_chunks(int64_t n);

// All parameters of one operator T = S·F·D·H (include/minnorm/srft.hpp:21-48)
// plus the derived per-chunk halo starts and the FFT-output selection map.
// The first `device_bytes` of `blob` are uploaded verbatim to the GPU.
struct SrftHost {
    int64_t n = 0, l = 0;
    int sampling = 0;        // MNB_WITHOUT_REPLACEMENT / MNB_WITH_REPLACEMENT
    int64_t max_mult = 1;    // max multiplicity of `sample` (lsq.cpp:31-39)
    int64_t max_span = 0;    // longest forward-chain scan of any chunk (chunk + halo + 1 steps)
    int64_t span_first = 0;  // the same over the Theta~ chain alone (the sketch's first H stage)
    bool first_derived = false;
    ChainChunks ch;

    // ---- blob layout (byte offsets) ----
    size_t off_d = 0, off_zeta = 0, off_zeta_tilde = 0;       // complex n
    size_t off_cssn = 0, off_cssn_tilde = 0;                   // (cos,sin) n (last unused)
    size_t off_perm = 0, off_perm_tilde = 0;                   // int32 n
    size_t off_sel = 0;                                        // int32 n: frequency -> slot or -1
    size_t off_halo = 0;                                       // int32 4*nchunks: fwd, fwd~, adj, adj~
    size_t off_sample = 0;                                     // int32 l
    size_t device_bytes = 0;
    size_t off_theta = 0, off_theta_tilde = 0;                 // host only: raw angles n-1
    size_t off_sample64 = 0;                                   // host only: int64 l
    size_t total_bytes = 0;
    std::vector<int32_t> dups;                                 // (slot, first_slot) pairs

    unsigned char* blob = nullptr;
    std::function<void(unsigned char*)> release;

    SrftHost() = default;
    SrftHost(const SrftHost&) = delete;
    SrftHost& operator=(const SrftHost&) = delete;
    ~SrftHost() { if (blob && release) release(blob); }

    template <class T> T* at(size_t off) { return reinterpret_cast<T*>(blob + off); }
    template <class T> const T* at(size_t off) const { return reinterpret_cast<const T*>(blob + off); }

    void layout();  // computes offsets from n, l
    // Derived data (halo starts, selection map, max multiplicity) from the fields.
    // derive_first: the part the sketch's first H stage needs (restart points of the
    // Theta~ chain); derive() runs it if it has not run, then the rest.
    void derive_first();
    void derive();
};

// Staged build.  The sketch's first H stage (Z~, Pi~, Theta~, Z: src/srft.cpp:52-55) needs
// only four of the eight parameter groups; a builder given a SrftStage draws those first and
// signals as soon as perm~, cos/sin(theta~), zeta~, zeta and their restart points are in the
// blob, while the other groups (d, theta, perm, sample) are still being drawn.  The values
// are the same streams in the same order: only the schedule changes.
struct SrftStage {
    std::mutex mu;
    std::condition_variable cv;
    int state = 0;  // 0 pending, 1 first half ready, 2 failed (the builder's future holds the error)
    void signal(int s) {
        {
            std::lock_guard<std::mutex> g(mu);
            if (state == 0) state = s;
        }
        cv.notify_all();
    }
    bool wait_first() {  // false: the build failed before the first half was ready
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return state != 0; });
        return state == 1;
    }
};

using BlobAlloc = std::function<unsigned char*(size_t)>;
using BlobFree = std::function<void(unsigned char*)>;

// build_srft(l, n, RandomStream(stream_seed), sampling) (src/srft.cpp:95-113)
// with the eight tagged substreams (srft.cpp:13-22) drawn concurrently and
// the cos/sin of finalize (srft.cpp:80-93) evaluated in parallel chunks.
// Throws mnb::Error(MNB_ERR_INVALID_ARGUMENT) like the reference.
// Run fn on a persistent background host thread (no per-solve thread creation).
std::future<void> host_async(std::function<void()> fn);

void build_srft_host(SrftHost& op, int64_t l, int64_t n, uint64_t stream_seed, int sampling,
                     const BlobAlloc& alloc, const BlobFree& release, int threads = 0, SrftStage* stage = nullptr);

}  // namespace mnb
