"""The hand-written sketch-QR kernels (csrc/k_cholqr.cu) against LAPACK, through the C ABI.

The reference factors its sketches with Eigen::HouseholderQR (src/solver.cpp:86, src/lsq.cpp:58)
and applies R by triangular solves (src/solver.cpp:93-96); the GPU path takes R from the Gram
matrix.  These tests pin each device stage on its own: the blocked Cholesky (R, potrf's info,
the rank rule of src/solver.cpp:25-33), the triangular inverse, and Step 2's z against the
Householder formula z = Q R^{-H} b, on ragged and block-aligned sizes.
"""
import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps


def crandn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def hermitian_pd(m, kappa, seed):
    rng = np.random.default_rng(seed)
    B = crandn(rng, 3 * m + 5, m)
    Q, _ = np.linalg.qr(B)
    V, _ = np.linalg.qr(crandn(rng, m, m))
    S = (Q * np.logspace(0, -np.log10(kappa), m)) @ V.conj().T
    return S, S.conj().T @ S


@pytest.mark.parametrize("m", [1, 2, 7, 31, 32, 33, 64, 65, 100, 256, 300, 1000])
def test_chol_upper_matches_lapack(ctx, m):
    _, G = hermitian_pd(m, 1e3, m)
    R, st = ctx.chol_upper(np.triu(G) + np.tril(np.full((m, m), 7.0 + 3j), -1))  # the lower triangle is not read
    want = sla.cholesky(G, lower=False)
    assert st["info"] == 0
    assert np.all(np.tril(R, -1) == 0)
    assert np.linalg.norm(R - want) <= 200 * EPS * np.linalg.cond(want) * np.linalg.norm(want)
    assert np.linalg.norm(R.conj().T @ R - G) <= 50 * m * EPS * np.linalg.norm(G)
    d = np.real(np.diag(R))
    assert st["dmin"] == pytest.approx(d.min(), rel=1e-12) and st["dmax"] == pytest.approx(d.max(), rel=1e-12)
    assert st["trace"] == pytest.approx(np.real(np.trace(G)), rel=1e-12)
    assert st["deficient"] == 0


def test_chol_upper_reports_the_failing_pivot(ctx):
    """potrf's info: 1 + index of the first non-positive pivot; NaN fails too."""
    m = 70
    _, G = hermitian_pd(m, 10.0, 3)
    v = np.zeros(m, complex)
    v[40] = 1.0
    Gbad = G - 2.0 * np.real(G[40, 40]) * np.outer(v, v)  # indefinite from pivot 40 on
    _, st = ctx.chol_upper(Gbad)
    assert 1 <= st["info"] <= 41
    try:
        sla.cholesky(Gbad, lower=False)
        raised = False
    except np.linalg.LinAlgError as e:
        raised = True
        assert str(st["info"]) in str(e)
    assert raised
    Gnan = G.copy()
    Gnan[10, 10] = np.nan
    _, st = ctx.chol_upper(Gnan)
    assert st["info"] == 11


def test_chol_upper_shift_and_rank_rule(ctx):
    m, l = 96, 400
    rng = np.random.default_rng(5)
    S = crandn(rng, l, m)
    S[:, 50] = S[:, 3] * (1.0 + 1e-15)  # a numerically dependent column
    G = S.conj().T @ S
    shift_factor = 11.0 * (l * m + m * (m + 1)) * EPS
    R, st = ctx.chol_upper(G, shift_factor=shift_factor, rank_rows=l)
    assert st["info"] == 0
    assert st["shift"] == pytest.approx(shift_factor * np.real(np.trace(G)), rel=1e-12)
    want = sla.cholesky(G + st["shift"] * np.eye(m), lower=False)
    assert np.linalg.norm(R - want) <= 1e-6 * np.linalg.norm(want)
    d = np.real(np.diag(R))
    assert st["deficient"] == int(np.sum(d < l * EPS * d.max()))


@pytest.mark.parametrize("m", [1, 5, 32, 33, 64, 96, 100, 129, 256, 500, 1024])
def test_trtri_upper_matches_lapack(ctx, m):
    rng = np.random.default_rng(100 + m)
    R = np.linalg.qr(crandn(rng, 2 * m + 3, m))[1]  # (a random triangle would be exponentially ill-conditioned)
    R = R * np.exp(1j * rng.uniform(0, 2 * np.pi, m))[:, None]  # complex diagonal
    X, xn = ctx.trtri_upper(R + np.tril(np.full((m, m), 9.0), -1))  # the lower triangle is not read
    want = sla.solve_triangular(R, np.eye(m), lower=False)
    assert np.all(np.tril(X, -1) == 0)
    assert np.linalg.norm(X - want) <= 100 * EPS * np.linalg.cond(R) * np.linalg.norm(want)
    assert np.linalg.norm(X @ R - np.eye(m)) <= 100 * m * EPS * np.linalg.cond(R)
    assert xn == pytest.approx(np.linalg.norm(want) ** 2, rel=1e-10)


@pytest.mark.parametrize("l,m,kappa", [(64, 16, 1e2), (256, 64, 1e3), (1024, 256, 1e6), (700, 100, 1e4), (4096, 1024, 1e4)])
def test_csne_step2_matches_householder(ctx, l, m, kappa):
    """z = Q R^{-H} b (src/solver.cpp:93-96) from the device-resident seminormal loop."""
    rng = np.random.default_rng(l + m)
    Qn, _ = np.linalg.qr(crandn(rng, l, m))
    Qm, _ = np.linalg.qr(crandn(rng, m, m))
    S = (Qn * np.logspace(0, -np.log10(kappa), m)) @ Qm.conj().T
    b = crandn(rng, m)
    z, st = ctx.csne_solve(S, b)
    Q, R = np.linalg.qr(S)
    want = Q @ sla.solve_triangular(R, b, trans="C", lower=False)
    assert st["accepted"]
    assert np.linalg.norm(z - want) <= 50 * EPS * kappa * np.linalg.norm(want)
    assert np.linalg.norm(S.conj().T @ z - b) <= 4 * np.sqrt(l) * EPS * np.linalg.norm(S) * np.linalg.norm(z)
    # (both are rounding-level quantities: the kernel's own value and numpy's agree in magnitude)
    assert st["residual"] <= 4 * np.sqrt(l) * EPS * np.linalg.norm(S) * np.linalg.norm(z)
    assert st["znorm"] == pytest.approx(np.linalg.norm(z), rel=1e-6)


def test_csne_rejects_an_ill_conditioned_sketch(ctx):
    """u cond(S)^2 >= 1: one Cholesky pass cannot carry Step 2; the solver then takes shifted CholeskyQR3."""
    rng = np.random.default_rng(9)
    l, m = 512, 64
    Qn, _ = np.linalg.qr(crandn(rng, l, m))
    Qm, _ = np.linalg.qr(crandn(rng, m, m))
    S = (Qn * np.logspace(0, -9, m)) @ Qm.conj().T
    _, st = ctx.csne_solve(S, crandn(rng, m))
    assert not st["accepted"]
