// Host SRFT parameter draw timings (run on the GPU box's host): one Fisher-Yates
// permutation, 1M sincos, and the full threaded operator draw at n = 2^20.
// g++ -O2 -std=c++20 -I paper_0905_4745_b200/csrc draw_bench.cpp paper_0905_4745_b200/csrc/host_srft.cpp -lpthread
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include "common_host.hpp"
#include "host_srft.hpp"

using namespace mnb;
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
    const int64_t n = 1 << 20;
    std::vector<int32_t> p(n);
    for (int rep = 0; rep < 3; ++rep) {
        RandomStream s(42 + rep);
        double t = now();
        s.permutation(p.data(), n);
        const double t_perm = now() - t;
        t = now();
        uint64_t acc = 0;
        for (int64_t i = 0; i < n; ++i) acc += s.next_u64();
        const double t_rng = now() - t;
        t = now();
        for (int64_t i = n; i > 1; --i) acc += s.next_u64() % uint64_t(i);
        const double t_mod = now() - t;
        std::vector<double> sn(n), cs(n);
        t = now();
        for (int64_t i = 0; i < n; ++i) ::sincos(double(i) * 1e-6, &sn[i], &cs[i]);
        const double t_sc = now() - t;
        std::vector<unsigned char> blob;
        SrftHost op;
        t = now();
        build_srft_host(op, 8192, n, 1234 + rep, MNB_WITHOUT_REPLACEMENT,
                        [&](size_t b) { blob.resize(b); return blob.data(); }, [](unsigned char*) {}, 16);
        const double t_op = now() - t;
        std::printf("perm %.2f ms  rng %.2f ms  rng+mod %.2f ms  sincos %.2f ms  operator(16 threads) %.2f ms  (%llu)\n",
                    t_perm * 1e3, t_rng * 1e3, t_mod * 1e3, t_sc * 1e3, t_op * 1e3, (unsigned long long)(acc & 1));
    }
    return 0;
}
