"""Pins the CPU oracle (oracle/) before it is trusted as the checker.

1. rng + per-vector kernels: bit-for-bit against the reference's OWN
   src/rng.cpp, src/kernels*.cpp compiled verbatim (oracle/_ref), and against
   the committed golden vectors (tests/golden/, made from oracle/_ref by
   tests/golden/make_golden.py).
2. fft / srft / lsq / solver: the known answers and dense oracles of the
   reference's own tests (tests/test_fft.cpp, test_srft.cpp, test_lsq.cpp,
   test_solver.cpp, test_support.hpp), restated here.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import minnorm_oracle as O
from tests.instances import make_instance

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
REF = O.ref_lib()
needs_ref = pytest.mark.skipif(REF is None, reason="oracle/_ref not built (needs /root/reference)")


def crandn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


# ---------------------------------------------------------------- dense oracles (tests/test_support.hpp)
def naive_dft(x):
    n = x.size
    j = np.arange(n)
    F = np.exp(-2j * np.pi * np.outer(j, j) / n) / np.sqrt(n)
    return F @ x


def dense_rotation_chain(theta):
    n = len(theta) + 1
    M = np.eye(n, dtype=complex)
    for k, t in enumerate(theta):
        R = np.eye(n, dtype=complex)
        R[k, k], R[k, k + 1], R[k + 1, k], R[k + 1, k + 1] = np.cos(t), np.sin(t), -np.sin(t), np.cos(t)
        M = M @ R
    return M


def dense_permutation(perm):
    n = len(perm)
    P = np.zeros((n, n), complex)
    P[np.arange(n), perm] = 1
    return P


def dense_h(op):
    return (dense_rotation_chain(op.field("theta")) @ dense_permutation(op.field("perm")) @ np.diag(op.field("zeta"))
            @ dense_rotation_chain(op.field("theta_tilde")) @ dense_permutation(op.field("perm_tilde"))
            @ np.diag(op.field("zeta_tilde")))


def dense_srft(op):
    n, l = op.n, op.l
    S = np.zeros((l, n), complex)
    S[np.arange(l), op.field("sample")] = 1
    F = np.exp(-2j * np.pi * np.outer(np.arange(n), np.arange(n)) / n) / np.sqrt(n)
    return S @ F @ np.diag(op.field("d")) @ dense_h(op)


def trivial_srft(l, n):
    return O.Srft.from_fields(l, n, np.ones(n), np.arange(l), np.zeros(n - 1), np.zeros(n - 1), np.arange(n),
                              np.arange(n), np.ones(n), np.ones(n))


# ---------------------------------------------------------------- rng vs reference build
SEEDS = [0, 1, 42, 7, 2**63 + 5, 0xFFFFFFFFFFFFFFFF]


@needs_ref
@pytest.mark.parametrize("seed", SEEDS)
def test_rng_streams_bit_exact_vs_reference_build(seed):
    import ctypes
    n = 4096
    a = np.zeros(n, np.uint64)
    REF.ref_rng_u64(seed, n, a.ctypes.data_as(ctypes.c_void_p))
    assert np.array_equal(a, O.rng_u64(seed, n))
    for kind, k in (("u01", 0), ("angle", 1), ("unit_circle", 2), ("sign", 3), ("complex_gaussian", 4)):
        cnt = 1000
        out = np.zeros(cnt * (2 if k in (2, 4) else 1))
        REF.ref_rng_draw(seed, k, cnt, out.ctypes.data_as(ctypes.c_void_p))
        ours = O.rng_draw(seed, kind, cnt)
        ours = ours.view(np.float64) if k in (2, 4) else ours
        assert np.array_equal(out.view(np.uint64), np.asarray(ours).view(np.uint64)), kind
    for tag in range(1, 20):
        assert int(REF.ref_derive_seed(seed, tag)) == O.derive_seed(seed, tag)


@needs_ref
@pytest.mark.parametrize("n", [1, 2, 3, 5, 64, 300, 100_003])
def test_permutation_and_sampling_bit_exact_vs_reference_build(n):
    import ctypes
    seed = 1000 + n
    p = np.zeros(n, np.int64)
    REF.ref_rng_permutation(seed, n, p.ctypes.data_as(ctypes.c_void_p))
    assert np.array_equal(p, O.rng_permutation(seed, n))
    for without in (1, 0):
        l = max(1, n // 3)
        s = np.zeros(l, np.int64)
        assert REF.ref_rng_sample(seed, l, n, without, s.ctypes.data_as(ctypes.c_void_p)) == 0
        assert np.array_equal(s, O.rng_sample(seed, l, n, bool(without)))


@needs_ref
@pytest.mark.parametrize("n", [2, 3, 5, 8, 64, 501, 4096])
def test_kernels_bit_exact_vs_reference_scalar_backend(n):
    """kernels_scalar.cpp restated: cmul, rotation_chain, fft_stage (tests/test_kernels.cpp)."""
    import ctypes
    assert REF.ref_kernels_select(b"scalar") == 0
    rng = np.random.default_rng(n)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    x, d = crandn(rng, n), crandn(rng, n)
    for conj in (0, 1):
        y1, y2 = np.zeros(n, complex), np.zeros(n, complex)
        REF.ref_cmul(P(y1), P(x), P(d), n, conj)
        O.lib().or_cmul(P(y2), P(x), P(d), n, conj)
        assert np.array_equal(y1, y2)
    th = rng.uniform(0, 2 * np.pi, n - 1)
    cs, sn = np.cos(th), np.sin(th)
    for adj in (0, 1):
        y1, y2 = x.copy(), x.copy()
        REF.ref_rotation_chain(P(y1), P(cs), P(sn), n, adj)
        O.lib().or_rotation_chain(P(y2), P(cs), P(sn), n, adj)
        assert np.array_equal(y1, y2)
    if n & (n - 1) == 0:
        gap = 1
        while gap < n:
            tw = np.exp(-1j * np.pi * np.arange(gap) / gap)
            y1, y2 = x.copy(), x.copy()
            REF.ref_fft_stage(P(y1), P(tw), n, gap, 0)
            O.lib().or_fft_stage(P(y2), P(tw), n, gap, 0)
            assert np.array_equal(y1, y2)
            gap *= 2


# ---------------------------------------------------------------- golden vectors
def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_golden_vectors():
    with open(os.path.join(GOLDEN, "rng_golden.json")) as f:
        g = json.load(f)
    for case in g["streams"]:
        s = case["seed"]
        assert [int(v) for v in O.rng_u64(s, len(case["u64"]))] == [int(v) for v in case["u64"]]
        assert O.rng_draw(s, "angle", len(case["angle"])).tolist() == case["angle"]
        uc = O.rng_draw(s, "unit_circle", len(case["unit_circle"]) // 2).view(np.float64).tolist()
        assert uc == case["unit_circle"]
        assert O.rng_permutation(s, 17).tolist() == case["perm17"]
        assert O.rng_sample(s, 5, 17, True).tolist() == case["sample_without"]
        assert O.rng_sample(s, 5, 17, False).tolist() == case["sample_with"]
        assert [O.derive_seed(s, t) for t in range(1, 13)] == case["derive"]


def test_srft_golden_vectors():
    with open(os.path.join(GOLDEN, "srft_golden.json")) as f:
        g = json.load(f)
    for case in g["operators"]:
        op = O.Srft.build(case["l"], case["n"], case["stream_seed"], True)
        for name, h in case["sha256"].items():
            assert _sha(op.field(name)) == h, name
        assert op.field("sample")[:4].tolist() == case["sample_head"]
        assert int(op.field("perm")[0]) == case["perm0"]


def test_survey_golden_values():
    """values derived from the verbatim rng.cpp, seed 42, substream(11)."""
    s11 = O.derive_seed(42, 11)
    op = O.Srft.build(8192, 1 << 20, s11)
    assert op.field("sample")[:4].tolist() == [413293, 426576, 565453, 361359]
    assert int(op.field("perm")[0]) == 499701
    d0 = op.field("d")[0]
    assert d0.real == 0.80575085203711838 and d0.imag == 0.59225464493025104
    op = O.Srft.build(4096, 1 << 17, s11)
    assert op.field("sample")[:4].tolist() == [20077, 113661, 74819, 56833]
    assert int(op.field("perm")[0]) == 87135


# ---------------------------------------------------------------- fft KATs (tests/test_fft.cpp)
def test_delta_transforms_to_flat_vector():
    e1 = np.zeros(4, complex)
    e1[0] = 1
    assert np.max(np.abs(O.dft(e1) - 0.5)) <= 1e-15


@pytest.mark.parametrize("n", [1, 2, 5, 8, 12, 31])
def test_ones_transform_to_sqrt_n_e1(n):
    y = O.dft(np.ones(n))
    assert abs(y[0] - np.sqrt(n)) <= 1e-12 * np.sqrt(n)
    assert np.all(np.abs(y[1:]) <= 1e-12)


def test_fast_matches_direct_formula_1_to_40():
    rng = np.random.default_rng(201)
    for n in range(1, 41):
        x = crandn(rng, n)
        assert np.linalg.norm(O.dft(x) - naive_dft(x)) <= 1e-13 * (1 + np.linalg.norm(x))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 16, 17, 100, 128, 1000, 1024])
def test_isometry_and_inverse(n):
    x = crandn(np.random.default_rng(203 + n), n)
    y = O.dft(x)
    assert abs(np.linalg.norm(y) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert np.linalg.norm(O.idft(y) - x) <= 1e-12 * np.linalg.norm(x)


# ---------------------------------------------------------------- srft KATs (tests/test_srft.cpp)
def test_trivial_operator_is_the_dft():
    n = 8
    op = trivial_srft(n, n)
    rng = np.random.default_rng(11)
    x = crandn(rng, n)
    assert np.linalg.norm(op.apply_h(x) - x) == 0.0
    assert np.linalg.norm(op.apply(x) - O.dft(x)) <= 1e-14 * np.linalg.norm(x)
    v = crandn(rng, n)
    assert np.linalg.norm(op.apply_adjoint(v) - O.idft(v)) <= 1e-14 * np.linalg.norm(v)


@pytest.mark.parametrize("n", [2, 3, 17, 64, 1000])
def test_h_is_unitary(n):
    op = O.Srft.build(1, n, O.derive_seed(13, n))
    x = crandn(np.random.default_rng(n), n)
    assert abs(np.linalg.norm(op.apply_h(x)) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)


def test_small_h_matches_explicit_factor_product():
    rng = np.random.default_rng(17)
    for rep in range(20):
        op = O.Srft.build(2, 3, O.derive_seed(17, rep))
        x = crandn(rng, 3)
        assert np.linalg.norm(op.apply_h(x) - dense_h(op) @ x) <= 1e-13 * np.linalg.norm(x)


@pytest.mark.parametrize("without", [True, False])
def test_fast_apply_matches_dense_factor_product(without):
    rng = np.random.default_rng(19)
    op = O.Srft.build(3, 8, O.derive_seed(19, int(not without)), without)
    T = dense_srft(op)
    x = crandn(rng, 8)
    assert np.linalg.norm(op.apply(x) - T @ x) <= 1e-13 * np.linalg.norm(x)
    v = crandn(rng, 3)
    assert np.linalg.norm(op.apply_adjoint(v) - T.conj().T @ v) <= 1e-13 * np.linalg.norm(v)
    M = crandn(rng, 8, 2)
    assert np.linalg.norm(op.sketch(np.conj(M).T.copy()) - T @ M) <= 1e-13 * np.linalg.norm(M)


@pytest.mark.parametrize("n", [6, 32, 100])
def test_adjoint_pairing_and_contraction(n):
    rng = np.random.default_rng(23 + n)
    l = n // 2
    op = O.Srft.build(l, n, O.derive_seed(23, n))
    x, v = crandn(rng, n), crandn(rng, l)
    lhs = np.vdot(v, op.apply(x))
    rhs = np.vdot(op.apply_adjoint(v), x)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(v)
    assert np.linalg.norm(op.apply(x)) <= np.linalg.norm(x) * (1 + 1e-12)
    assert abs(np.linalg.norm(op.apply_adjoint(v)) - np.linalg.norm(v)) <= 1e-12 * np.linalg.norm(v)


def test_with_replacement_duplicates_accumulate():
    op = O.Srft.from_fields(2, 4, np.ones(4), [1, 1], np.zeros(3), np.zeros(3), np.arange(4), np.arange(4),
                            np.ones(4), np.ones(4), without=False)
    expect = np.zeros(4, complex)
    expect[1] = 3
    assert np.linalg.norm(op.apply_adjoint(np.array([1, 2], complex)) - O.idft(expect)) <= 1e-14


def test_materialized_rows_orthonormal():
    op = O.Srft.build(5, 16, O.derive_seed(31, 3))
    T = np.stack([op.apply(e) for e in np.eye(16, dtype=complex)], axis=1)
    assert np.linalg.norm(T @ T.conj().T - np.eye(5)) <= 1e-12


# ---------------------------------------------------------------- lsq / solver (tests/test_lsq.cpp, test_solver.cpp)
def test_lsq_excess_below_tau_against_dense_reference():
    A, _ = make_instance(8, 64, 1e3, seed=47)
    c = crandn(np.random.default_rng(305), 64)
    tau = 1e-10
    sol = O.solve_least_squares(A, c, 32, tau, 300, 49)
    B = A.conj().T
    best = np.linalg.norm(B @ O.least_squares_qr(A, c) - c) ** 2
    got = np.linalg.norm(B @ sol.y - c) ** 2
    assert sol.converged
    assert got - best <= tau * best + 1e-24 * np.linalg.norm(c) ** 2
    assert sol.achieved_excess <= tau


def test_lsq_consistent_system():
    A, _ = make_instance(8, 96, 10.0, seed=41)
    B = A.conj().T
    c = B @ crandn(np.random.default_rng(301), 8)
    sol = O.solve_least_squares(A, c, 32, 1e-12, 300, 43)
    assert sol.converged
    assert np.linalg.norm(B @ sol.y - c) <= 1e-10 * np.linalg.norm(c)


def test_solver_orthonormal_rows_and_single_row():
    A = np.zeros((2, 16), complex)
    A[0, 0] = A[1, 1] = 1
    rep = O.solve_randomized(A, np.array([1, 1], complex), epsilon=1e-8)
    want = np.zeros(16, complex)
    want[:2] = 1
    assert np.linalg.norm(rep.x - want) <= 1e-8 * np.linalg.norm(want)
    assert rep.residual_norm <= 1e-10 and rep.lsq_converged
    A = np.zeros((1, 16), complex)
    A[0, 0], A[0, 1] = 3, 4
    want = np.zeros(16, complex)
    want[0], want[1] = 0.6, 0.8
    assert np.linalg.norm(O.solve_randomized(A, np.array([5.0 + 0j]), epsilon=1e-9).x - want) <= 1e-9
    assert np.linalg.norm(O.solve_classical(A, np.array([5.0 + 0j])) - want) <= 1e-14


def test_solver_tracks_exact_minimal_norm_solution():
    A, b = make_instance(64, 1024, 1e3, seed=1)
    p = O.solve_svd(A, b)
    assert np.linalg.norm(O.solve_classical(A, b) - p) <= 1e-12 * 1e3 * np.linalg.norm(p)
    rep = O.solve_randomized(A, b, epsilon=1e-12)
    assert np.linalg.norm(rep.x - p) <= 1e-11 * np.linalg.norm(p)
    assert rep.lsq_converged


def test_solver_tau_and_errors():
    A, b = make_instance(4, 64, 1e2, seed=109)
    rep = O.solve_randomized(A, b)
    assert rep.sketch_size == 16
    assert rep.lsq_tau == pytest.approx(1e-12 * 16.0 / (4.0 * 64.0))
    A, b = make_instance(4, 12, 10.0, seed=97)
    with pytest.raises(O.ConfigError):
        O.solve_randomized(A, b)
    with pytest.raises(O.ConfigError):
        O.solve_randomized(A, b, sketch_size=4)
    with pytest.raises(O.ConfigError):
        O.solve_randomized(A, b, sketch_size=8, epsilon=2.0)
    with pytest.raises(O.ConfigError):
        O.solve_randomized(A, b, sketch_size=8, alpha=1.0)


@pytest.mark.parametrize("real", [False, True])
def test_exact_minnorm_against_svd_and_pivoted_qr(real):
    """The extended-precision exact p (oracle.exact_minnorm, the yardstick of the full-size
    parity campaign) agrees with the reference's SVD oracle (src/solver.cpp:148-156) at a
    well-conditioned desk size, and at kappa = 1e6 it sits far below the float64 floor: the
    pivoted-QR solution (src/solver.cpp:130-146) is ~u*kappa away from it, not more."""
    A, b = make_instance(64, 1024, 10.0, seed=211, real=real)
    p, hist = O.exact_minnorm(A, b)
    assert np.linalg.norm(p - O.solve_svd(A, b)) <= 1e-14 * np.linalg.norm(p)
    assert hist[-1] <= 1e-15
    A, b = make_instance(128, 8192, 1e6, seed=212, real=real)
    p, _ = O.exact_minnorm(A, b)
    p2, _ = O.exact_minnorm(A, b, chunk=1000)  # chunking / threading does not change the answer
    assert np.linalg.norm(p - p2) <= 1e-13 * np.linalg.norm(p)
    e_qr = np.linalg.norm(O.solve_classical(A, b) - p) / np.linalg.norm(p)
    assert 1e-13 < e_qr <= 10 * O.EPS * 1e6


# ---- tests/acceptance.cpp criteria against the oracle (pins generate_instance + solve_randomized)
def test_acceptance_oracle_equivalence_200_trials():
    """acceptance.cpp:50-75: 200 generated instances, randomized (eps 1e-6) vs SVD <= 1e-6."""
    worst = 0.0
    for trial in range(200):
        m = 2 + trial % 7
        n = m * (8 << (trial % 4))
        kappa = 1e3 if trial % 2 else 1.0
        gen = O.generate_instance(m, n, kappa, 9000 + trial)
        assert np.allclose(np.linalg.svd(gen.A, compute_uv=False)[[0, -1]], [1.0, 1.0 / kappa], rtol=1e-12)
        x = O.solve_randomized(gen.A, gen.b, sketch_size=4 * m, epsilon=1e-6, seed=O.derive_seed(9000 + trial, 77),
                               threads=1).x
        p = O.solve_svd(gen.A, gen.b)
        worst = max(worst, np.linalg.norm(x - p) / np.linalg.norm(p))
    assert worst <= 1e-6


def test_acceptance_table2_eps_r_oracle():
    """acceptance.cpp:77-90 (3 of the 10 trials on the CPU): eps_r <= 1e-13 at 128 x 16384, l = 512."""
    gen = O.generate_instance(128, 16384, 1e6, O.derive_seed(1001, 100))
    eps = O.bench_epsilon(1e6, 128, 512)
    assert eps == pytest.approx(1e-8)
    for trial in range(3):
        rep = O.solve_randomized(gen.A, gen.b, sketch_size=512, epsilon=eps, seed=O.derive_seed(1001, 1000 + trial))
        assert O.normalized_error(rep.x, gen.p_true, 1e6) <= 1e-13
