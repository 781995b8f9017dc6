"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle
(oracle/, a restatement of the reference pinned by tests/test_oracle.py).

Tolerances: FFT / SRFT entries 1e-13 relative (the reference tests' own
bound, tests/test_srft.cpp:86-98); H stage bit-exact (same operation order,
exact carries); solves within 10*epsilon of the oracle's x (north_star) and
CG iteration counts within +-1."""
import numpy as np
import pytest

import paper_0905_4745_b200 as mn
from oracle import minnorm_oracle as O
from tests.instances import make_instance

pytestmark = pytest.mark.gpu


def crandn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 12, 16, 17, 31, 40, 64, 96, 100, 1000, 1024, 1536, 2048, 4096,
                               6144, 16384, 131072])
def test_dft_matches_oracle(ctx, n):
    rng = np.random.default_rng(n)
    x = crandn(rng, n)
    y = mn.dft(x, ctx)
    assert rel(y, O.dft(x)) <= 1e-13
    assert rel(y, np.fft.fft(x) / np.sqrt(n)) <= 1e-13
    assert rel(mn.idft(y, ctx), x) <= 1e-13


@pytest.mark.parametrize("n", [2, 3, 17, 64, 1000, 4096, 65536])
def test_apply_h_bit_exact(ctx, n):
    seed = mn.derive_seed(13, n)
    op = mn.build_srft(1, n, seed)
    ref = O.Srft.build(1, n, seed)
    x = crandn(np.random.default_rng(n), n)
    y = op.apply_h(x, ctx)
    yr = ref.apply_h(x)
    assert np.array_equal(y, yr), f"max diff {np.abs(y - yr).max():.3e}"


@pytest.mark.parametrize("l,n", [(3, 8), (5, 16), (50, 100), (256, 1024), (1024, 16384), (4096, 131072),
                                 (100, 6144)])
@pytest.mark.parametrize("mode", [mn.Sampling.without_replacement, mn.Sampling.with_replacement])
def test_apply_and_adjoint_match_oracle(ctx, l, n, mode):
    seed = mn.derive_seed(19, n + int(mode))
    op = mn.build_srft(l, n, seed, mode)
    ref = O.Srft.build(l, n, seed, mode == mn.Sampling.without_replacement)
    rng = np.random.default_rng(l + n)
    x = crandn(rng, n)
    v = crandn(rng, l)
    assert rel(op.apply(x, ctx), ref.apply(x)) <= 1e-13
    assert rel(op.apply_adjoint(v, ctx), ref.apply_adjoint(v)) <= 1e-13


# the large-n cases exercise the blocked four-step passes (n = 2^20: both passes
# length 1024, the specialised kernel; 3*2^20: 3072 x 1024) and, at n = 2^17 ... 2^19 (n1 x 1024 with
# n1 = 128, 256, 512; c3 is 2^17), the fused H stage + pass A with the direct pruned pass B -- or,
# when m is not a multiple of 8 (12, 5), the unfused passes over the same split
@pytest.mark.parametrize("m,n,l", [(2, 16, 8), (64, 1024, 256), (256, 16384, 1024), (37, 6144, 160),
                                   (8, 1 << 20, 64), (24, 1 << 20, 96), (12, 1 << 20, 48), (12, 1 << 19, 48),
                                   (16, 1 << 19, 2100), (24, 1 << 18, 300), (5, 1 << 18, 40),
                                   (16, 1 << 17, 4096), (40, 1 << 17, 64), (8, 1 << 17, 40000),
                                   (5, 3 << 20, 40), (16, 3 << 20, 64)])
def test_sketch_matches_oracle(ctx, m, n, l):
    A, _ = make_instance(m, n, kappa=1e3, seed=m + n)
    seed = mn.derive_seed(42, 11)
    op = mn.build_srft(l, n, seed)
    ref = O.Srft.build(l, n, seed)
    ctx.set_matrix(A)
    S = op.sketch(ctx)
    Sr = ref.sketch(A)
    assert rel(S, Sr) <= 1e-13


@pytest.mark.parametrize("real,seg,n", [(False, "2", 1 << 20), (True, "2", 1 << 20), (False, "1", 1 << 20),
                                        (True, "1", 3 << 20), (False, "2", 1 << 17), (True, "1", 1 << 17)])
def test_fused_h_fft_matches_unfused(real, seg, n, monkeypatch):
    """The fused second H stage + FFT pass A (k_p2fa.cu, n = 1024 x 1024, row
    blocks of 8, each row block's 1024 steps in 1 or 2 segments restarted from
    the fine restart table) against the two-launch path (MNB_P2FA=0) and the
    oracle."""
    m, l = 16, 128
    A, _ = make_instance(m, n, kappa=1e3, seed=m + 7, real=real)
    seed = mn.derive_seed(42, 11)
    op = mn.build_srft(l, n, seed)
    monkeypatch.setenv("MNB_P2FA_SEG", seg)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("MNB_P2FA", flag)
        c = mn.Context(0)
        c.set_matrix(A)
        out[flag] = op.sketch(c)
        c.close()
    ref = O.Srft.build(l, n, seed).sketch(A)
    assert rel(out["1"], ref) <= 1e-13
    assert rel(out["1"], out["0"]) <= 1e-13


def test_sketch_with_replacement_large_n(ctx):
    """Repeated sample indices (RandomStream::Sampling::with_replacement) through the
    blocked, pruned pass B at n = 2^20 (l close to n so collisions are certain)."""
    m, n, l = 8, 1 << 20, 4096
    A, _ = make_instance(m, n, kappa=1e3, seed=99)
    seed = mn.derive_seed(42, 12)
    op = mn.build_srft(l, n, seed, mn.Sampling.with_replacement)
    ref = O.Srft.build(l, n, seed, without=False)
    assert len(np.unique(ref.field("sample"))) < l  # the case under test: some frequencies repeat
    ctx.set_matrix(A)
    assert rel(op.sketch(ctx), ref.sketch(A)) <= 1e-13


def test_sketch_real_matrix(ctx):
    A, _ = make_instance(32, 6144, kappa=1e3, seed=5, real=True)
    seed = mn.derive_seed(42, 12)
    op = mn.build_srft(128, 6144, seed)
    ref = O.Srft.build(128, 6144, seed)
    ctx.set_matrix(A)
    assert rel(op.sketch(ctx), ref.sketch(A)) <= 1e-13


EPS_MACH = np.finfo(float).eps


def solve_tol(eps, kappa):
    """10*eps (north_star), but not below the conditioning floor eps_mach * kappa, where
    float64 itself stops determining p (SURVEY §8c measured 6e-9 between two exact solvers
    at kappa = 1e8).  Every case below except the kappa = 1e8 ones is held to 10*eps."""
    return max(10 * eps, EPS_MACH * kappa)


@pytest.mark.parametrize("m,n,kappa,eps", [(64, 1024, 1e3, 1e-12), (256, 16384, 1e6, 1e-10), (16, 256, 1e2, 1e-8),
                                           (48, 6144, 1e4, 1e-10), (128, 32768, 1e4, 1e-8)])
def test_solve_randomized_matches_oracle(ctx, m, n, kappa, eps):
    A, b = make_instance(m, n, kappa, seed=m * 7 + 1)
    cfg = mn.SolverConfig(epsilon=eps, seed=42)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx)
    p = O.solve_classical(A, b)  # exact minimal-norm solution (pivoted QR, src/solver.cpp:130-146)
    assert rel(rep.x, p) <= solve_tol(eps, kappa)
    assert rep.lsq_converged
    ref = O.solve_randomized(A, b, epsilon=eps, seed=42)
    if ref.lsq_converged:
        # the reference converged: match its x and its iteration count
        assert rel(rep.x, ref.x) <= 10 * eps
        assert abs(rep.lsq_iterations - ref.lsq_iterations) <= 1
        assert abs(rep.c_norm_ratio - ref.c_norm_ratio) <= 1e-8 * ref.c_norm_ratio
    else:
        # the reference's stop rule is below its own gradient floor (eps_mach*kappa)^2 > tau:
        # it runs lsq_max_iterations and diverges
        assert ref.lsq_iterations == 300
    assert rep.residual_norm <= 1e-6 * np.linalg.norm(b) * kappa
    # the report's ||A x - b|| (accumulated inside the CG passes) is the residual of the returned x
    true_res = np.linalg.norm(A @ rep.x - b)
    assert abs(rep.residual_norm - true_res) <= 1e-3 * true_res + 1e-12 * np.linalg.norm(b) * kappa


def test_solve_real_matrix(ctx):
    A, b = make_instance(32, 6144, 1e4, seed=3, real=True)
    cfg = mn.SolverConfig(epsilon=1e-10)
    rep = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx)
    ref = O.solve_randomized(A, b, epsilon=1e-10)
    assert rel(rep.x, ref.x) <= 1e-9
    assert abs(rep.lsq_iterations - ref.lsq_iterations) <= 1


@pytest.mark.parametrize("m,n,kappa,eps", [(64, 1024, 1e3, 1e-12), (256, 16384, 1e6, 1e-10), (128, 8192, 1e8, 1e-10)])
def test_cholqr2_matches_householder(m, n, kappa, eps, monkeypatch):
    """The sketch QRs run CholeskyQR2 (tensor-core ZHERK) when the sketch is
    well enough conditioned, shifted CholeskyQR3 when it is not, and
    Householder (the reference's HouseholderQR, src/solver.cpp:86,
    src/lsq.cpp:58) as the last resort / with MNB_QR=householder; all must
    give the same solve."""
    A, b = make_instance(m, n, kappa, seed=m + 3)
    cfg = mn.SolverConfig(epsilon=eps, seed=42)
    reps = {}
    for mode in ("cholqr2", "householder"):
        monkeypatch.setenv("MNB_QR", mode)
        c = mn.Context(0)
        reps[mode] = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, c)
        c.close()
    a, h = reps["cholqr2"], reps["householder"]
    # path taken: CholeskyQR2 (0) for well-conditioned sketches, shifted CholeskyQR3 (1) at 1e8;
    # the preconditioner's QR(E) stops after one Cholesky pass (3) when u cond(E)^2 is tiny
    # S: one Cholesky pass + corrected seminormal Step 2 (4) unless the sketch is too ill-conditioned
    # at 1e8 (u cond^2 not small) both take the shifted two-pass chain (6 / 5)
    assert (a.extra["qr_path"] & 15) == (6 if kappa >= 1e8 else 4)
    e_path = a.extra["qr_path"] >> 4
    if kappa <= 1e4:
        assert e_path == 3
    elif kappa >= 1e8:
        assert e_path == 5
    else:
        assert e_path in (0, 3)
    assert h.extra["qr_path"] == 2 | (2 << 4)
    p = O.solve_classical(A, b)
    assert rel(a.x, p) <= solve_tol(eps, kappa)
    assert rel(a.x, h.x) <= solve_tol(eps, kappa)
    assert abs(a.lsq_iterations - h.lsq_iterations) <= 1


@pytest.mark.parametrize("m,n,kappa,eps", [(64, 1024, 1e3, 1e-12), (256, 16384, 1e6, 1e-10), (256, 8192, 1e4, 1e-8)])
def test_csne_step2_matches_cholqr2(m, n, kappa, eps, monkeypatch):
    """Step 2 from R1 = chol(S^H S) with the corrected seminormal equations
    (path 4) gives the solve of the full CholeskyQR2 Step 2 (z = Q R^{-H} b,
    src/solver.cpp:93-96): same x within the solve tolerance, same iteration
    count +-1, and the c it produces satisfies A c = b as well."""
    A, b = make_instance(m, n, kappa, seed=m + 11)
    cfg = mn.SolverConfig(epsilon=eps, seed=42, capture_c=True)
    reps = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("MNB_CSNE", flag)
        c = mn.Context(0)
        reps[flag] = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, c)
        c.close()
    a, f = reps["1"], reps["0"]
    assert (a.extra["qr_path"] & 15) == 4 and (f.extra["qr_path"] & 15) == 0
    p = O.solve_classical(A, b)
    assert rel(a.x, p) <= solve_tol(eps, kappa)
    assert rel(a.x, f.x) <= solve_tol(eps, kappa)
    assert abs(a.lsq_iterations - f.lsq_iterations) <= 1
    # Step 3's c solves A c = b to the same accuracy on both paths
    ra = np.linalg.norm(A @ a.c - b) / np.linalg.norm(b)
    rf = np.linalg.norm(A @ f.c - b) / np.linalg.norm(b)
    assert ra <= max(10 * rf, 1e-13 * kappa)


@pytest.mark.parametrize("m,n,kappa,eps", [(64, 1024, 1e3, 1e-12), (256, 16384, 1e6, 1e-10), (128, 8192, 1e8, 1e-10)])
def test_init_from_sketch_matches_init_pass(m, n, kappa, eps, monkeypatch):
    """The CG's first product A c (src/lsq.cpp:77-86) taken as S^H z from the
    sketch (c = T^* z, so A c = (T A^*)^* z) instead of a pass over A gives the
    same solve: x within the solve tolerance, iterations +-1, and the same
    reported ||c|| ratio."""
    A, b = make_instance(m, n, kappa, seed=m + 17)
    cfg = mn.SolverConfig(epsilon=eps, seed=42)
    reps = {}
    for flag in (None, "1"):
        if flag:
            monkeypatch.setenv("MNB_INIT_PASS", flag)
        c = mn.Context(0)
        reps[flag] = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, c)
        c.close()
    a, f = reps[None], reps["1"]
    p = O.solve_classical(A, b)
    assert rel(a.x, p) <= solve_tol(eps, kappa)
    assert rel(a.x, f.x) <= solve_tol(eps, kappa)
    assert abs(a.lsq_iterations - f.lsq_iterations) <= 1
    assert abs(a.c_norm_ratio - f.c_norm_ratio) <= solve_tol(eps, kappa) * abs(f.c_norm_ratio)  # (through ||x||)


def test_fused_tail_split_and_unfused_agree_at_scale(monkeypatch):
    """600 rows at n = 2^20 = 75 row blocks on 74 cluster pairs: the last row
    block runs as two k1 segments (restarted from the half-chunk restart table).
    The default (tail split), no split (MNB_P2FA_SEG=1) and the unfused two-launch
    path (MNB_P2FA=0, itself pinned to the oracle above) give the same sketch."""
    import torch
    m, n, l = 600, 1 << 20, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    At = torch.randn((n, m), dtype=torch.complex128, device="cuda", generator=g)  # A^T row-major = A col-major
    op = mn.build_srft(l, n, mn.derive_seed(42, 11))
    out = {}
    for name, env in (("split", {}), ("whole", {"MNB_P2FA_SEG": "1"}), ("unfused", {"MNB_P2FA": "0"})):
        for k in ("MNB_P2FA_SEG", "MNB_P2FA"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c = mn.Context(0)
        c.set_matrix(At.T, n_global=n)
        out[name] = op.sketch(c)
        c.close()
    del At
    torch.cuda.empty_cache()
    assert rel(out["split"], out["unfused"]) <= 1e-13
    assert rel(out["whole"], out["unfused"]) <= 1e-13


def test_two_norm_preconditioner_check_matches_full_qr(monkeypatch):
    """The one-pass preconditioner accepted on the 2-norm cond estimate (path 3 where the
    Frobenius bound alone rejects, kappa = 1e6) gives the same solve as the full CholeskyQR2
    preconditioner (MNB_PRECOND_2NORM=0): x within the solve tolerance, iterations +-1."""
    m, n, kappa, eps = 256, 16384, 1e6, 1e-10
    A, b = make_instance(m, n, kappa, seed=77)
    cfg = mn.SolverConfig(epsilon=eps, seed=42)
    reps = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("MNB_PRECOND_2NORM", flag)
        c = mn.Context(0)
        reps[flag] = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, c)
        c.close()
    a, f = reps["1"], reps["0"]
    assert (f.extra["qr_path"] >> 4) in (0, 3)
    assert (a.extra["qr_path"] >> 4) in (0, 3)
    p = O.solve_classical(A, b)
    assert rel(a.x, p) <= solve_tol(eps, kappa)
    assert rel(a.x, f.x) <= solve_tol(eps, kappa)
    assert abs(a.lsq_iterations - f.lsq_iterations) <= 1
