// generate_instance (include/minnorm/bench.hpp; src/bench.cpp:46-74): the reference front end's
// synthetic instance A = U diag(sigma) V^H with U (m x m) and V (n x m) orthonormalised complex
// Gaussians, sigma_j = kappa^{-j/(m-1)}, p_true = V w with w_j = +-1/sqrt(m), b = A p_true.
// Host side (it feeds the `gen` and `bench` subcommands of the CLI); the draws follow the
// reference's RandomStream substreams 21 / 22 / 23 (src/bench.cpp:16) in the same order.
#include <cmath>
#include <complex>
#include <vector>

#include "host_srft.hpp"
#include "common_host.hpp"

namespace mnb {
namespace {

using cplx = std::complex<double>;

// src/bench.cpp:18-23: complex_gaussian() in column-major order.
std::vector<cplx> gaussian_matrix(RandomStream s, int64_t rows, int64_t cols) {
    std::vector<cplx> X(static_cast<size_t>(rows * cols));
    for (auto& x : X) {
        double ri[2];
        s.complex_gaussian(ri);
        x = cplx(ri[0], ri[1]);
    }
    return X;
}

// src/bench.cpp:26-37: modified Gram-Schmidt, two projection sweeps per column.
void orthonormalize_columns(std::vector<cplx>& X, int64_t rows, int64_t cols) {
    for (int64_t j = 0; j < cols; ++j) {
        cplx* v = X.data() + j * rows;
        for (int sweep = 0; sweep < 2; ++sweep)
            for (int64_t i = 0; i < j; ++i) {
                const cplx* q = X.data() + i * rows;
                cplx d = 0.0;
                for (int64_t k = 0; k < rows; ++k) d += std::conj(q[k]) * v[k];
                for (int64_t k = 0; k < rows; ++k) v[k] -= d * q[k];
            }
        double nrm = 0.0;
        for (int64_t k = 0; k < rows; ++k) nrm += std::norm(v[k]);
        nrm = std::sqrt(nrm);
        if (!(nrm > 0.0)) throw Error(MNB_ERR_INTERNAL, "orthonormalize_columns: degenerate Gaussian draw");
        for (int64_t k = 0; k < rows; ++k) v[k] /= nrm;
    }
}

}  // namespace

void generate_instance(int64_t m, int64_t n, double kappa, uint64_t stream_seed, double* A_out, double* b_out,
                       double* p_out) {
    if (m < 2) throw Error(MNB_ERR_DIMENSION, "generate_instance: m must be at least 2");
    if (m >= n) throw Error(MNB_ERR_DIMENSION, "generate_instance: need m < n");
    if (!(kappa >= 1.0)) throw Error(MNB_ERR_DIMENSION, "generate_instance: kappa must be >= 1");
    const RandomStream stream(stream_seed);
    std::vector<cplx> U = gaussian_matrix(stream.substream(21), m, m);
    orthonormalize_columns(U, m, m);
    std::vector<cplx> V = gaussian_matrix(stream.substream(22), n, m);
    orthonormalize_columns(V, n, m);
    std::vector<double> sigma(static_cast<size_t>(m));
    for (int64_t j = 0; j < m; ++j) sigma[size_t(j)] = std::pow(kappa, -double(j) / double(m - 1));
    // A = (U diag(sigma)) V^H, column-major m x n
    cplx* A = reinterpret_cast<cplx*>(A_out);
    for (int64_t c = 0; c < n; ++c)
        for (int64_t r = 0; r < m; ++r) {
            cplx acc = 0.0;
            for (int64_t k = 0; k < m; ++k) acc += U[size_t(k * m + r)] * sigma[size_t(k)] * std::conj(V[size_t(k * n + c)]);
            A[c * m + r] = acc;
        }
    RandomStream signs = stream.substream(23);
    std::vector<cplx> w(static_cast<size_t>(m));
    const double scale = 1.0 / std::sqrt(double(m));
    for (auto& x : w) x = signs.sign() * scale;
    cplx* p = reinterpret_cast<cplx*>(p_out);
    for (int64_t r = 0; r < n; ++r) {
        cplx acc = 0.0;
        for (int64_t k = 0; k < m; ++k) acc += V[size_t(k * n + r)] * w[size_t(k)];
        p[r] = acc;
    }
    cplx* b = reinterpret_cast<cplx*>(b_out);
    for (int64_t r = 0; r < m; ++r) {
        cplx acc = 0.0;
        for (int64_t c = 0; c < n; ++c) acc += A[c * m + r] * p[c];
        b[r] = acc;
    }
}

}  // namespace mnb
