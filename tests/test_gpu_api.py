"""The reference's solver / least-squares contracts, run through the GPU path.

Each test mirrors a TEST_CASE of /root/reference/proj/tests/test_solver.cpp or
tests/test_lsq.cpp (cited per test): known answers, error behaviour (the
exception types of include/minnorm/errors.hpp), determinism, reporting.
Instances come from tests/instances.py (the BASELINE construction) or are
written out as in the reference test.
"""
import numpy as np
import pytest

import paper_0905_4745_b200 as mn
from oracle import minnorm_oracle as O
from tests.instances import make_instance

pytestmark = pytest.mark.gpu


def crandn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def conditioned_tall(n, m, kappa, seed):
    """B = Q_n diag(sigma) Q_m^H, n x m, singular values log-spaced 1 -> 1/kappa."""
    rng = np.random.default_rng(seed)
    Qn, _ = np.linalg.qr(crandn(rng, n, m))
    Qm, _ = np.linalg.qr(crandn(rng, m, m))
    return (Qn * np.logspace(0, -np.log10(kappa), m)) @ Qm.conj().T


# ------------------------------------------------------------ test_solver.cpp
def test_orthonormal_row_analog(ctx):
    """test_solver.cpp:45-63: 2 x 16 orthonormal rows force x = (1, 1, 0, ...)."""
    A = np.zeros((2, 16), complex)
    A[0, 0] = A[1, 1] = 1.0
    b = np.array([1.0, 1.0], complex)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(epsilon=1e-8), ctx)
    want = np.zeros(16, complex)
    want[:2] = 1.0
    assert np.linalg.norm(rep.x - want) <= 1e-8 * np.linalg.norm(want)
    assert rep.residual_norm <= 1e-10
    assert rep.lsq_converged


def test_single_row_projects_onto_the_row(ctx):
    """test_solver.cpp:65-75: A = (3, 4, 0, ...), b = 5 -> x = (0.6, 0.8, 0, ...)."""
    A = np.zeros((1, 16), complex)
    A[0, 0], A[0, 1] = 3.0, 4.0
    b = np.array([5.0], complex)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(epsilon=1e-9), ctx)
    want = np.zeros(16, complex)
    want[0], want[1] = 0.6, 0.8
    assert np.linalg.norm(rep.x - want) <= 1e-9


def test_conditioned_instance_tracks_exact_solution(ctx):
    """test_solver.cpp:77-90 (l = 16, eps = 1e-6, seed 73; healthy c_norm_ratio)."""
    A, b = make_instance(4, 32, 1e3, seed=71)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(sketch_size=16, epsilon=1e-6, seed=73), ctx)
    p = O.solve_svd(A, b)
    assert np.linalg.norm(rep.x - p) <= 1e-6 * np.linalg.norm(p)
    assert rep.lsq_converged
    assert rep.c_norm_ratio <= 1.5


def test_zero_rhs_short_circuits(ctx):
    """test_solver.cpp:118-128 (src/solver.cpp:68-73)."""
    A, _ = make_instance(3, 48, 1e2, seed=95)
    rep = mn.solve_randomized(mn.ProblemInstance(A, np.zeros(3, complex)), mn.SolverConfig(), ctx)
    assert np.linalg.norm(rep.x) == 0.0
    assert rep.residual_norm == 0.0


@pytest.mark.parametrize("kw", [dict(), dict(sketch_size=4), dict(sketch_size=12),
                                dict(sketch_size=8, epsilon=2.0), dict(sketch_size=8, alpha=1.0)])
def test_bad_configuration_raises_config_error(ctx, kw):
    """test_solver.cpp:130-145: l outside (m, n), eps outside (0, 1), alpha <= 1."""
    A, b = make_instance(4, 12, 1e1, seed=97)
    with pytest.raises(mn.ConfigError):
        mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(**kw), ctx)


def test_dimension_and_finiteness_preconditions(ctx):
    """test_solver.cpp:147-160 and ProblemInstance::validate (src/solver.cpp:37-48)."""
    rng = np.random.default_rng(99)
    with pytest.raises(mn.DimensionError):  # not underdetermined
        mn.solve_randomized(mn.ProblemInstance(crandn(rng, 4, 4), crandn(rng, 4)), mn.SolverConfig(), ctx)
    with pytest.raises(mn.DimensionError):  # b length
        mn.solve_randomized(mn.ProblemInstance(crandn(rng, 2, 8), crandn(rng, 3)), mn.SolverConfig(), ctx)
    bad = crandn(rng, 2, 64)
    bad[1, 3] = np.nan
    with pytest.raises(mn.DimensionError):  # non-finite A (checked on the device while sketching)
        mn.solve_randomized(mn.ProblemInstance(bad, crandn(rng, 2)), mn.SolverConfig(), ctx)
    with pytest.raises(mn.DimensionError):  # non-finite b
        b = crandn(rng, 2)
        b[0] = np.inf
        mn.solve_randomized(mn.ProblemInstance(crandn(rng, 2, 64), b), mn.SolverConfig(), ctx)


def test_rank_deficiency_is_reported(ctx):
    """test_solver.cpp:162-174: a rank-1 2 x 16 matrix."""
    rng = np.random.default_rng(101)
    A = np.zeros((2, 16), complex)
    A[0] = crandn(rng, 16)
    A[1] = 2.0 * A[0]
    b = np.array([1.0, 2.0], complex)
    with pytest.raises(mn.RankDeficiencyError) as ei:
        mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(sketch_size=8), ctx)
    assert ei.value.deficient_columns() >= 1


def test_unconverged_subsolver_is_reported_not_thrown(ctx):
    """test_solver.cpp:176-185: lsq_max_iterations = 1."""
    A, b = make_instance(6, 96, 1e5, seed=103)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(epsilon=1e-9, lsq_max_iterations=1), ctx)
    assert not rep.lsq_converged
    assert np.all(np.isfinite(rep.x))


def test_fixed_seed_is_bitwise_reproducible_and_captures_c(ctx):
    """test_solver.cpp:187-204: same bits of x and c across runs; A c = b; c only on request."""
    A, b = make_instance(4, 64, 1e3, seed=105)
    cfg = mn.SolverConfig(seed=107, capture_c=True)
    r1 = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx)
    r2 = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx)
    assert r1.x.tobytes() == r2.x.tobytes()
    assert r1.c is not None and r1.c.size == A.shape[1]
    assert r1.c.tobytes() == r2.c.tobytes()
    assert np.linalg.norm(A @ r1.c - b) <= 1e-10 * 1e3 * np.linalg.norm(b)
    cfg.capture_c = False
    assert mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx).c is None


def test_report_fields(ctx):
    """test_solver.cpp:206-213: step timings, sketch size, lsq_tau = eps^2 l / (alpha n)."""
    A, b = make_instance(4, 64, 1e2, seed=109)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(), ctx)
    assert all(t >= 0.0 for t in rep.step_seconds)
    assert rep.sketch_size == 16
    assert rep.lsq_tau == pytest.approx(1e-12 * 16.0 / (4.0 * 64.0))


def test_with_replacement_sampling_solve(ctx):
    """RandomStream::Sampling::with_replacement through the whole solve (dup > 1 in the stop rule)."""
    A, b = make_instance(16, 256, 1e2, seed=111)
    cfg = mn.SolverConfig(epsilon=1e-10, sampling=mn.Sampling.with_replacement)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx)
    ref = O.solve_randomized(A, b, epsilon=1e-10, without=False)
    p = O.solve_classical(A, b)
    assert np.linalg.norm(rep.x - p) <= 1e-8 * np.linalg.norm(p)
    assert abs(rep.lsq_iterations - ref.lsq_iterations) <= 1


# --------------------------------------------------------------- test_lsq.cpp
def lsq(B, c, l, tau, seed, ctx, max_iterations=300):
    return mn.solve_least_squares(B, c, mn.LsqConfig(sketch_size=l, tau=tau, stream_seed=seed,
                                                     max_iterations=max_iterations), ctx)


def test_lsq_orthonormal_columns_reduce_to_adjoint_projection(ctx):
    """test_lsq.cpp:42-50."""
    rng = np.random.default_rng(303)
    B, _ = np.linalg.qr(crandn(rng, 64, 6))
    c = crandn(rng, 64)
    sol = lsq(B, c, 24, 1e-14, 45, ctx)
    assert np.linalg.norm(sol.y - B.conj().T @ c) <= 1e-10 * np.linalg.norm(c)


@pytest.mark.parametrize("trial", range(6))
def test_lsq_excess_below_tau(ctx, trial):
    """test_lsq.cpp:52-82: got - best <= tau best across conditions and tolerances."""
    rng = np.random.default_rng(400 + trial)
    m = 2 + trial
    n = 16 * m
    kappa = 10.0 ** (trial % 7)
    B = conditioned_tall(n, m, kappa, 500 + trial)
    c = B @ crandn(rng, m) + 0.25 * crandn(rng, n)
    c /= np.linalg.norm(c)
    tau = 10.0 ** (-4.0 - 4.0 * (trial % 3))
    sol = lsq(B, c, 4 * m, tau, 600 + trial, ctx)
    y_best = np.linalg.lstsq(B, c, rcond=None)[0]
    best = np.linalg.norm(B @ y_best - c) ** 2
    got = np.linalg.norm(B @ sol.y - c) ** 2
    assert got - best <= tau * best + 1e-24
    ref = O.solve_least_squares(np.asfortranarray(B.conj().T), c, 4 * m, tau, stream_seed=600 + trial)
    assert abs(sol.iterations - ref.iterations) <= 1


def test_lsq_residual_norms_never_increase(ctx):
    """test_lsq.cpp:84-92."""
    rng = np.random.default_rng(307)
    B = conditioned_tall(128, 12, 1e4, 51)
    c = B @ crandn(rng, 12) + 0.5 * crandn(rng, 128)
    sol = lsq(B, c, 48, 1e-14, 53, ctx)
    assert len(sol.residual_norms) >= 2
    for k in range(1, len(sol.residual_norms)):
        assert sol.residual_norms[k] <= sol.residual_norms[k - 1] * (1.0 + 1e-12)


def test_lsq_fixed_seed_is_bitwise_reproducible(ctx):
    """test_lsq.cpp:94-100."""
    rng = np.random.default_rng(309)
    B = conditioned_tall(80, 6, 1e2, 55)
    c = crandn(rng, 80)
    y1 = lsq(B, c, 24, 1e-10, 57, ctx).y
    y2 = lsq(B, c, 24, 1e-10, 57, ctx).y
    assert y1.tobytes() == y2.tobytes()


@pytest.mark.parametrize("m,n", [(192, 4096), (1032, 8192)])
def test_pinned_host_matrix_pipelined_copy_matches(ctx, m, n):
    """A page-locked host A takes the MNB_HOST_ASYNC path (row-slab H2D overlapped with both
    sketches); the solve must equal the one from a pageable (eagerly copied) A.  (m >= 1024:
    seven equal slabs and a short, here ragged, last one.)"""
    torch = pytest.importorskip("torch")
    A, b = make_instance(m, n, 1e3, seed=113)
    pinned = torch.empty((A.shape[1], A.shape[0]), dtype=torch.complex128, pin_memory=True)
    pinned.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
    A_pinned = pinned.numpy().T  # column-major view of page-locked memory
    cfg = mn.SolverConfig(epsilon=1e-10, capture_c=True)
    r_pin = mn.solve_randomized(mn.ProblemInstance(A_pinned, b), cfg, ctx)
    r_page = mn.solve_randomized(mn.ProblemInstance(np.asfortranarray(A), b), cfg, ctx)
    # the sketches are bit-identical; the pipelined path forms E's Gram block by block as the slabs
    # land (one ZGEMM per slab) where the eager path takes one ZHERK, so R' -- and the CG iterates --
    # agree to rounding.  For m > 1024 it forms S's Gram the same way, so there c agrees to rounding
    # too; below that QR(S) takes its own ZHERK and c is bit-identical.
    if m <= 1024:
        assert r_pin.c.tobytes() == r_page.c.tobytes()
    else:
        assert np.linalg.norm(r_pin.c - r_page.c) <= 1e-12 * np.linalg.norm(r_page.c)
    assert r_pin.lsq_iterations == r_page.lsq_iterations
    assert np.linalg.norm(r_pin.x - r_page.x) <= 1e-12 * np.linalg.norm(r_page.x)
    # a later call on the same context sees the resident matrix
    op = mn.build_srft(4 * m, n, mn.derive_seed(42, 11))
    ctx.set_matrix(A_pinned, deferred=True)
    S1 = op.sketch(ctx)
    ctx.set_matrix(np.asfortranarray(A))
    assert np.array_equal(S1, op.sketch(ctx))


# ---- solve_classical (src/solver.cpp:130-146) on the GPU ----------------------------------
@pytest.mark.parametrize("m,n,kappa,path", [(64, 1024, 1e3, 0), (256, 16384, 1e6, 0), (128, 8192, 1e8, 1),
                                            (16, 6000, 1e2, 0)])
def test_solve_classical_matches_oracle(ctx, m, n, kappa, path):
    """The device classical solver (Gram + corrected seminormal equations, or Householder QR
    of A^H when u cond(A)^2 is not small) against the oracle's pivoted-QR solve_classical:
    the same minimal-norm x to within the problem's conditioning (1e-13 kappa), a residual at
    the rounding level, and the path the header documents."""
    A, b = make_instance(m, n, kappa, seed=m + 21)
    x, rep = mn.solve_classical(mn.ProblemInstance(A, b), ctx, report=True)
    p = O.solve_classical(A, b)
    assert np.linalg.norm(x - p) / np.linalg.norm(p) <= max(1e-14 * kappa, 1e-12)
    assert rep.path == path
    assert abs(rep.residual_norm - np.linalg.norm(A @ x - b)) <= 1e-6 * np.linalg.norm(b) + 1e-3 * rep.residual_norm
    assert rep.residual_norm <= 1e-12 * np.linalg.norm(A, 2) * np.linalg.norm(x) * np.sqrt(n)


def test_solve_classical_real_matrix(ctx):
    """Real A (the c5 type): the Gram path with DSYRK, same x as the oracle."""
    A, b = make_instance(48, 4096, 1e3, seed=8, real=True)
    x, rep = mn.solve_classical(mn.ProblemInstance(A, b), ctx, report=True)
    p = O.solve_classical(A.astype(np.complex128), b)
    assert rep.path == 0
    assert np.linalg.norm(x - p) / np.linalg.norm(p) <= 1e-11


def test_solve_classical_zero_rhs_and_errors(ctx):
    """b = 0 gives x = 0 (src/solver.cpp:134); a rank-deficient A raises RankDeficiencyError;
    a wrong-length b raises DimensionError (ProblemInstance::validate)."""
    A, b = make_instance(32, 512, 1e2, seed=4)
    x = mn.solve_classical(mn.ProblemInstance(A, np.zeros(32, np.complex128)), ctx)
    assert np.all(x == 0)
    Ad = A.copy()
    Ad[5] = Ad[3]  # two equal rows: rank m - 1
    with pytest.raises(mn.RankDeficiencyError):
        mn.solve_classical(mn.ProblemInstance(Ad, b), ctx)
    with pytest.raises(mn.DimensionError):
        mn.solve_classical(mn.ProblemInstance(A, b[:5]), ctx)


def test_solve_classical_rank_handling_real_and_ill_conditioned(ctx):
    """real A and very ill-conditioned A reach the Householder fallback (path 1) and
    are either solved or reported as RankDeficiencyError with the deficient-column count -- the
    rank rule applied to the singular values of R (rank-revealing), never UNSUPPORTED."""
    # full rank, kappa = 1e9: the Gram path cannot take it, path 1 solves it (complex and real)
    for real in (False, True):
        A, b = make_instance(48, 4096, 1e9, seed=12, real=real)
        x, rep = mn.solve_classical(mn.ProblemInstance(A, b), ctx, report=True)
        p = O.solve_classical(A.astype(np.complex128), b)
        assert rep.path == 1
        assert np.linalg.norm(x - p) / np.linalg.norm(p) <= 1e-14 * 1e9
    # two dependent rows, one of them perturbed below the n eps threshold: rank m - 2
    A, b = make_instance(32, 2048, 1e2, seed=13, real=True)
    Ad = A.copy()
    Ad[7] = Ad[3]
    Ad[9] = 2.0 * Ad[4] + 1e-15 * Ad[0]
    with pytest.raises(mn.RankDeficiencyError) as e:
        mn.solve_classical(mn.ProblemInstance(Ad, b), ctx)
    assert e.value.deficient_columns() == 2
    assert O.deficient_count(np.linalg.qr(np.conj(Ad.astype(np.complex128)).T, mode="r"), 2048) >= 1


def test_solve_classical_agrees_with_randomized(ctx):
    """The paper's comparison (Tables 1-4): the randomized solve matches the classical one to
    its epsilon."""
    A, b = make_instance(128, 4096, 1e4, seed=9)
    cfg = mn.SolverConfig(epsilon=1e-10, seed=42)
    xr = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx).x
    xc = mn.solve_classical(mn.ProblemInstance(A, b), ctx)
    assert np.linalg.norm(xr - xc) / np.linalg.norm(xc) <= 10 * cfg.epsilon


def test_apply_adjoint_matrix(ctx):
    """mnb_apply_adjoint_matrix: x = A^H y and A x from one fused pass (Step 5 of the solve,
    src/solver.cpp:118-125) against numpy; complex and real A."""
    for real in (False, True):
        A, _ = make_instance(40, 3000, 1e2, seed=31, real=real)
        rng = np.random.default_rng(3)
        y = rng.standard_normal(40) + 1j * rng.standard_normal(40)
        ctx.set_matrix(A)
        x, ax = mn.apply_adjoint_matrix(y, ctx, with_ax=True)
        xr = A.conj().T @ y
        assert np.linalg.norm(x - xr) <= 1e-13 * np.linalg.norm(xr)
        assert np.linalg.norm(ax - A @ xr) <= 1e-13 * np.linalg.norm(A @ xr)
        with pytest.raises(mn.DimensionError):
            mn.apply_adjoint_matrix(y[:5], ctx)


# -------------------------------------------------- staged draw of T (host_srft.hpp SrftStage)
_STAGED_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_0905_4745_b200 as mn
from tests.instances import make_instance
A, b = make_instance(24, 65536, 1e3, seed=311)
ctx = mn.Context(0)
r = mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(seed=313, capture_c=True), ctx)
print(hashlib.sha256(r.x.tobytes()).hexdigest(), hashlib.sha256(r.c.tobytes()).hexdigest(), r.lsq_iterations)
"""


def test_staged_draw_gives_the_same_bits():
    """The staged draw / upload of T (first H stage's groups first, the rest behind P1) only
    reschedules src/srft.cpp:95-113: x and c equal the one-shot draw's bit for bit.  (The switches
    are read once per process, hence the subprocesses; n = 2^16 is where staging starts.)"""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"MNB_STAGED_DRAW": "0"}):
        e = dict(os.environ)
        e.update(env)
        p = subprocess.run([sys.executable, "-c", _STAGED_SCRIPT.format(root=root)], capture_output=True, text=True,
                           env=e, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(p.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]
