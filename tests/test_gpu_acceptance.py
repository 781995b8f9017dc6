"""The reference's acceptance criteria (tests/acceptance.cpp) through the GPU path.

* criterion_oracle_equivalence (acceptance.cpp:50-75): 200 generated instances
  (m = 2..8, n = 8m..64m, kappa 1 or 1e3, generate_instance of src/bench.cpp:46-74,
  restated in oracle.generate_instance), the randomized solve at epsilon 1e-6
  against the SVD solution: relative error <= 1e-6 on every trial.
* criterion_table2 / criterion_table4 (acceptance.cpp:77-104): run_benchmark's
  rows (src/bench.cpp:86-127) at the paper's Table 2 / Table 4 sizes, kappa 1e6,
  10 trials each, epsilon = bench_epsilon: the kappa-normalised error
  eps_r = ||x - p_true|| / (kappa ||p_true||) <= 1e-13.
"""
import numpy as np
import pytest

import paper_0905_4745_b200 as mn
from oracle import minnorm_oracle as O

pytestmark = pytest.mark.gpu


def test_oracle_equivalence_200_trials(ctx):
    eps = 1e-6
    worst, failures = 0.0, 0
    for trial in range(200):
        m = 2 + trial % 7
        n = m * (8 << (trial % 4))
        kappa = 1e3 if trial % 2 else 1.0
        gen = O.generate_instance(m, n, kappa, 9000 + trial)
        cfg = mn.SolverConfig(sketch_size=4 * m, alpha=4.0, epsilon=eps, seed=mn.derive_seed(9000 + trial, 77))
        x = mn.solve_randomized(mn.ProblemInstance(gen.A, gen.b), cfg, ctx).x
        p = O.solve_svd(gen.A, gen.b)
        rel = float(np.linalg.norm(x - p) / np.linalg.norm(p))
        worst = max(worst, rel)
        failures += rel > eps
    assert failures == 0, f"failures {failures}/200, worst rel err {worst:.2e}"


def run_benchmark_row(ctx, m, n, l, idx, base_seed, trials=10, kappa=1e6):
    """src/bench.cpp:86-127 for one grid row: eps_r over `trials` seeds."""
    gen = O.generate_instance(m, n, kappa, O.derive_seed(base_seed, 100 + idx))
    eps = O.bench_epsilon(kappa, m, l, 4.0)
    epsr = 0.0
    for trial in range(trials):
        cfg = mn.SolverConfig(sketch_size=l, alpha=4.0, epsilon=eps,
                              seed=O.derive_seed(base_seed, 1000 * (idx + 1) + trial))
        rep = mn.solve_randomized(mn.ProblemInstance(gen.A, gen.b), cfg, ctx)
        epsr = max(epsr, O.normalized_error(rep.x, gen.p_true, kappa))
    return epsr


def test_table2_eps_r(ctx):
    assert run_benchmark_row(ctx, 128, 16384, 512, 0, 1001) <= 1e-13


def test_table4_eps_r(ctx):
    worst = max(run_benchmark_row(ctx, 256, 4096, 1024, 0, 1003), run_benchmark_row(ctx, 256, 8192, 1024, 1, 1003))
    assert worst <= 1e-13
