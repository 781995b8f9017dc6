// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
// A C-ABI shim over the reference's OWN Eigen-free sources, which
// oracle/Makefile (target `ref`) compiles verbatim from /root/reference:
//   proj/src/rng.cpp, proj/src/kernels.cpp, proj/src/kernels_scalar.cpp,
//   proj/src/kernels_avx2.cpp   ->  oracle/_ref/libminnorm_ref.so
// The rest of the reference (fft/srft/lsq/solver) needs Eigen3, which is not
// in this image, so it is unbuildable here.
// Used only by tests/ to pin oracle/minnorm_oracle.cpp and the product's
// host parameter generator bit-for-bit against the reference itself.
#include <complex>
#include <cstdint>
#include <cstring>
#include <vector>

#include "minnorm/kernels.hpp"
#include "minnorm/rng.hpp"

using minnorm::RandomStream;
using C = std::complex<double>;

extern "C" {
uint64_t ref_derive_seed(uint64_t seed, uint64_t tag) { return RandomStream(seed).derive_seed(tag); }
void ref_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
    RandomStream r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}
void ref_rng_draw(uint64_t seed, int kind, int64_t count, double* out) {
    RandomStream r(seed);
    for (int64_t i = 0; i < count; ++i) {
        switch (kind) {
            case 0: out[i] = r.uniform01(); break;
            case 1: out[i] = r.uniform_angle(); break;
            case 2: { C z = r.unit_circle(); out[2 * i] = z.real(); out[2 * i + 1] = z.imag(); } break;
            case 3: out[i] = r.sign(); break;
            case 4: { C z = r.complex_gaussian(); out[2 * i] = z.real(); out[2 * i + 1] = z.imag(); } break;
        }
    }
}
void ref_rng_permutation(uint64_t seed, int64_t n, int64_t* out) {
    RandomStream r(seed);
    auto p = r.permutation(size_t(n));
    for (int64_t i = 0; i < n; ++i) out[i] = int64_t(p[size_t(i)]);
}
int ref_rng_sample(uint64_t seed, int64_t l, int64_t n, int without, int64_t* out) {
    try {
        RandomStream r(seed);
        auto p = r.sample_indices(size_t(l), size_t(n),
                                  without ? RandomStream::Sampling::without_replacement
                                          : RandomStream::Sampling::with_replacement);
        for (int64_t i = 0; i < l; ++i) out[i] = int64_t(p[size_t(i)]);
        return 0;
    } catch (...) { return -1; }
}
// backend: "scalar" or "avx2"; returns 0 if the backend could be selected.
int ref_kernels_select(const char* name) { return minnorm::kernels::select(name) ? 0 : -1; }
void ref_cmul(double* y, const double* x, const double* d, int64_t n, int conj) {
    const auto& ops = minnorm::kernels::active();
    (conj ? ops.cmul_conj : ops.cmul)((C*)y, (const C*)x, (const C*)d, size_t(n));
}
void ref_rotation_chain(double* x, const double* cs, const double* sn, int64_t n, int adjoint) {
    minnorm::kernels::active().rotation_chain((C*)x, cs, sn, size_t(n), adjoint != 0);
}
void ref_fft_stage(double* x, const double* tw, int64_t n, int64_t gap, int conj_tw) {
    minnorm::kernels::active().fft_stage((C*)x, (const C*)tw, size_t(n), size_t(gap), conj_tw != 0);
}
}
