"""The distributed (NCCL) code path on one B200, and the multi-slab sketch.

`Context.distributed` with world_size 1 builds a one-rank NCCL communicator and
takes exactly the multi-GPU path of solver.cu / srft_gpu.cu: the one all-to-all
of A into row blocks (redistribute_rows, shared by both sketches), the sketch
allgather, the finiteness allreduce and the per-iteration CG allreduce.  With
one rank every exchange is an identity, so the solve must reproduce the
single-GPU solve.  (This environment has one GPU per call; ranks that wait on
one another must not share a GPU, so world sizes above 1 are covered by the
gloo tests of the same exchange table, tests/test_dist_gloo.py.)

The multi-slab sketch (Ms < m, taken at c5 where A is 96 GiB) is forced at
small m with MNB_SLAB_ROWS and checked against the default slab and the oracle.
"""
import os

import numpy as np
import pytest

import paper_0905_4745_b200 as mn
from oracle import minnorm_oracle as O
from tests.instances import make_instance

pytestmark = pytest.mark.gpu


def _rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.fixture(scope="module")
def dctx():
    c = mn.Context.distributed(0, 0, 1, mn.Context.nccl_unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("real", [False, True])
def test_world1_nccl_solve_matches_single_gpu(ctx, dctx, real):
    A, b = make_instance(96, 8192, 1e4, seed=21, real=real)
    cfg = mn.SolverConfig(epsilon=1e-10, capture_c=True)
    single = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, ctx)
    dist = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, dctx, n_global=A.shape[1])
    assert dist.extra["world_size"] == 1
    assert dist.extra["redistribute_seconds"] > 0.0  # the all-to-all ran (once: both sketches share it)
    assert dist.lsq_iterations == single.lsq_iterations
    assert dist.lsq_converged
    # the one-GPU solve of an L2-resident A runs the persistent CG kernel, the distributed one the
    # multi-kernel loop: the same iterates up to the order of the partial sums
    assert _rel(dist.x, single.x) <= 1e-11
    assert _rel(dist.c, single.c) <= 1e-13
    ref = O.solve_randomized(A, b, epsilon=1e-10, seed=42)
    assert _rel(dist.x, ref.x) <= 10 * cfg.epsilon
    assert abs(dist.lsq_iterations - ref.lsq_iterations) <= 1


def test_world1_nccl_sketch_classical_and_adjoint(ctx, dctx):
    A, b = make_instance(64, 4096, 1e3, seed=5)
    op = mn.build_srft(256, 4096, mn.derive_seed(42, 11))
    dctx.set_shard(A, n_global=A.shape[1])
    S_d = op.sketch(dctx)
    ctx.set_matrix(A)
    S_s = op.sketch(ctx)
    assert np.array_equal(S_d, S_s)
    x_d = mn.solve_classical(mn.ProblemInstance(A, b), dctx, n_global=A.shape[1])
    x_s = mn.solve_classical(mn.ProblemInstance(A, b), ctx)
    assert _rel(x_d, x_s) <= 1e-13
    y = np.random.default_rng(1).standard_normal(64) + 0j
    xd, axd = mn.apply_adjoint_matrix(y, dctx, with_ax=True)
    xs, axs = mn.apply_adjoint_matrix(y, ctx, with_ax=True)
    assert np.array_equal(xd, xs) and _rel(axd, axs) <= 1e-14


def test_world1_nccl_classical_householder_path(ctx, dctx):
    """The TSQR form of the Householder fallback (path 1) through the distributed code path
    (allgather of R_J, QR of the stack) equals the one-GPU path; rank deficiency is reported."""
    A, b = make_instance(40, 3000, 1e9, seed=17)
    x_d, rep_d = mn.solve_classical(mn.ProblemInstance(A, b), dctx, report=True, n_global=A.shape[1])
    x_s, rep_s = mn.solve_classical(mn.ProblemInstance(A, b), ctx, report=True)
    assert rep_d.path == 1 and rep_s.path == 1
    assert _rel(x_d, x_s) <= 1e-10
    Ad = A.copy()
    Ad[6] = Ad[2]
    with pytest.raises(mn.RankDeficiencyError):
        mn.solve_classical(mn.ProblemInstance(Ad, b), dctx, n_global=A.shape[1])


def test_distributed_shard_validation(dctx):
    A, b = make_instance(16, 512, 1e2, seed=2)
    fresh = mn.Context.distributed(0, 0, 1, mn.Context.nccl_unique_id())
    try:
        with pytest.raises(ValueError):  # no global column count yet
            mn.solve_randomized(mn.ProblemInstance(A, b), mn.SolverConfig(), fresh)
        with pytest.raises(mn.DimensionError):  # shard width != mnb_shard_columns(n_global)
            mn.solve_randomized(mn.ProblemInstance(A[:, :500], b), mn.SolverConfig(), fresh, n_global=512)
    finally:
        fresh.close()


def test_redistribute_plan_covers_the_matrix():
    for world in (1, 2, 3, 8):
        for rank in range(world):
            m, n = 37, 1001
            p = mn.redistribute_plan(m, n, world, rank)
            my_rows = mn.shard_columns(m, world, rank)[1]
            my_cols = mn.shard_columns(n, world, rank)[1]
            assert p[:, 1].sum() == m and p[:, 4].sum() == n
            assert list(p[:, 2]) == list(np.concatenate([[0], np.cumsum(p[:-1, 1] * my_cols)]))
            assert list(p[:, 5]) == list(p[:, 3] * my_rows)


def _with_env(var, val, fn):
    old = os.environ.get(var)
    os.environ[var] = val
    try:
        return fn()
    finally:
        if old is None:
            os.environ.pop(var, None)
        else:
            os.environ[var] = old


@pytest.mark.parametrize("n", [1 << 20, 3 << 20])
def test_multislab_sketch_matches_single_slab_and_oracle(n):
    """The c5 sketch runs in row slabs (Ms < m).  Force 8/16-row slabs on 48 rows and compare
    with the one-slab sketch (bit for bit) and the oracle (1e-13)."""
    rng = np.random.default_rng(3)
    m, l = 48, 192
    real = n % 3 == 0
    A = rng.standard_normal((m, n)) if real else (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    A = np.asfortranarray(A)
    op = mn.build_srft(l, n, mn.derive_seed(42, 11))

    def sketch():
        c = mn.Context(0)
        try:
            c.set_matrix(A)
            return op.sketch(c)
        finally:
            c.close()

    one = sketch()
    for rows in ("8", "16"):
        multi = _with_env("MNB_SLAB_ROWS", rows, sketch)
        assert np.array_equal(multi, one), f"slab of {rows} rows differs from the single slab"
    ref = O.Srft.build(l, n, O.derive_seed(42, 11)).sketch(A[:8], threads=os.cpu_count())
    assert _rel(one[:, :8], ref) <= 1e-13


def test_multislab_solve_matches_default():
    A, b = make_instance(64, 3 << 16, 1e4, seed=9, real=True)
    cfg = mn.SolverConfig(epsilon=1e-10)

    def solve():
        c = mn.Context(0)
        try:
            return mn.solve_randomized(mn.ProblemInstance(A, b), cfg, c)
        finally:
            c.close()

    d = solve()
    s = _with_env("MNB_SLAB_ROWS", "16", solve)
    # the sketches are bit-identical; with several slabs E's Gram is built block by block (one ZGEMM
    # per slab) where one slab takes a ZHERK, so R' and the CG iterates agree to rounding
    assert s.lsq_iterations == d.lsq_iterations
    assert _rel(s.x, d.x) <= 1e-12


def test_error_mid_solve_leaves_the_context_usable():
    """A solve that raises after both sketches were queued (rank deficiency, with the multi-slab
    sketch and its per-slab Gram hook active, and QR(E) on the helper thread) must leave the context
    clean: the next solve on it equals a solve on a fresh context."""
    A, b = make_instance(48, 3 << 16, 1e3, seed=4, real=True)
    Ad = A.copy()
    Ad[5] = Ad[3]
    cfg = mn.SolverConfig(epsilon=1e-10)

    def run():
        c = mn.Context(0)
        try:
            with pytest.raises(mn.RankDeficiencyError):
                mn.solve_randomized(mn.ProblemInstance(Ad, b), cfg, c)
            after = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, c)
        finally:
            c.close()
        c = mn.Context(0)
        try:
            fresh = mn.solve_randomized(mn.ProblemInstance(A, b), cfg, c)
        finally:
            c.close()
        return after, fresh

    after, fresh = _with_env("MNB_SLAB_ROWS", "16", run)
    assert after.lsq_converged and after.lsq_iterations == fresh.lsq_iterations
    assert np.array_equal(after.x, fresh.x)
