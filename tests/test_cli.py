"""The minnorm_b200 command-line front end: the cases of the reference's
tests/test_cli.cpp:46-138 restated (pipeline, determinism, exit codes, bench CSV,
MINNORM_SEED), plus selftest and its --corrupt-dft fault hook (src/selftest.cpp:239).
Host-only subcommands run in the CPU suite; anything that solves runs under -m gpu."""
import os
import subprocess

import numpy as np
import pytest

import paper_0905_4745_b200 as mn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_0905_4745_b200", "bin", "minnorm_b200")


def run(args, env=None, cwd=None):
    e = dict(os.environ)
    e.pop("MINNORM_SEED", None)
    e.update(env or {})
    p = subprocess.run([CLI] + args, capture_output=True, text=True, env=e, cwd=cwd, timeout=600)
    return p.returncode, p.stdout, p.stderr


# ------------------------------------------------------------------ CPU (host only)
def test_gen_writes_the_instance_and_matches_the_library(tmp_path):
    prefix = str(tmp_path / "inst")
    rc, out, _ = run(["gen", "--m", "4", "--n", "64", "--kappa", "1e3", "--seed", "5", "--out", prefix])
    assert rc == 0 and '"subcommand": "gen"' in out and '"seed": 5' in out
    A = mn.read_matrix_market(prefix + "_A.mtx")
    g = mn.generate_instance(4, 64, 1e3, 5)
    assert np.array_equal(A, g.A)
    assert np.array_equal(mn.read_vector_market(prefix + "_b.mtx"), g.b)
    assert np.array_equal(mn.read_vector_market(prefix + "_p.mtx"), g.p_true)
    assert np.allclose(np.linalg.svd(A, compute_uv=False)[[0, -1]], [1.0, 1e-3], rtol=1e-12)


def test_oracle_residual_mode(tmp_path):
    prefix = str(tmp_path / "inst")
    assert run(["gen", "--m", "3", "--n", "48", "--seed", "9", "--out", prefix])[0] == 0
    rc, out, _ = run(["oracle", prefix + "_A.mtx", prefix + "_b.mtx", "--residual", "--solution", prefix + "_p.mtx"])
    assert rc == 0 and '"relative_residual"' in out
    assert run(["oracle", prefix + "_A.mtx", prefix + "_b.mtx", "--residual"])[0] == 4  # needs --solution


def test_exit_codes_without_a_solve(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix array complex general\n2 2\n1 0\nnot-a-number 0\n")
    prefix = str(tmp_path / "inst")
    assert run(["gen", "--m", "2", "--n", "24", "--seed", "3", "--out", prefix])[0] == 0
    assert run(["solve", str(bad), prefix + "_b.mtx"])[0] == 2                       # parse
    assert run(["solve", str(tmp_path / "missing.mtx"), prefix + "_b.mtx"])[0] == 2
    assert run(["baseline", prefix + "_A.mtx", prefix + "_A.mtx"])[0] == 3           # b is a matrix
    assert run(["solve", prefix + "_A.mtx", prefix + "_b.mtx", "--sampling", "sometimes"])[0] == 4
    assert run(["gen", "--m", "10", "--n", "4", "--out", str(tmp_path / "x")])[0] == 3  # bad dims
    assert run(["totally-unknown-subcommand"])[0] == 4
    assert run(["solve", "--unknown-flag", "1"])[0] == 4


def test_minnorm_seed_is_the_fallback_seed(tmp_path):
    rc, out, _ = run(["gen", "--m", "2", "--n", "24", "--out", str(tmp_path / "env")], env={"MINNORM_SEED": "77"})
    assert rc == 0 and '"seed": 77' in out
    assert run(["gen", "--m", "2", "--n", "24", "--out", str(tmp_path / "env")], env={"MINNORM_SEED": "x"})[0] == 4


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_gen_solve_baseline_oracle_pipeline(tmp_path):
    prefix = str(tmp_path / "inst")
    assert run(["gen", "--m", "4", "--n", "64", "--kappa", "1e3", "--seed", "5", "--out", prefix])[0] == 0
    x = str(tmp_path / "x.mtx")
    rc, out, err = run(["solve", prefix + "_A.mtx", prefix + "_b.mtx", "--seed", "7", "--epsilon", "1e-8", "--out", x])
    assert rc == 0, err
    assert '"residual_norm"' in out and '"lsq_converged": true' in out
    rc, out, _ = run(["oracle", prefix + "_A.mtx", prefix + "_b.mtx", "--residual", "--solution", x])
    assert rc == 0 and '"relative_residual"' in out
    xb, xo = str(tmp_path / "xb.mtx"), str(tmp_path / "xo.mtx")
    assert run(["baseline", prefix + "_A.mtx", prefix + "_b.mtx", "--out", xb])[0] == 0
    assert run(["oracle", prefix + "_A.mtx", prefix + "_b.mtx", "--out", xo])[0] == 0
    p = mn.read_vector_market(prefix + "_p.mtx")
    for f, tol in ((x, 1e-6), (xb, 1e-11), (xo, 1e-11)):
        v = mn.read_vector_market(f)
        assert np.linalg.norm(v - p) / np.linalg.norm(p) <= tol, f


@pytest.mark.gpu
def test_repeated_seeded_solves_are_byte_identical(tmp_path):
    prefix = str(tmp_path / "inst")
    assert run(["gen", "--m", "3", "--n", "48", "--seed", "9", "--out", prefix])[0] == 0
    xs = [str(tmp_path / f"x{k}.mtx") for k in range(3)]
    for f, seed in zip(xs, ("11", "11", "12")):
        assert run(["solve", prefix + "_A.mtx", prefix + "_b.mtx", "--seed", seed, "--out", f])[0] == 0
    b1 = open(xs[0], "rb").read()
    assert b1 and b1 == open(xs[1], "rb").read()
    assert open(xs[2], "rb").read() != b1


@pytest.mark.gpu
def test_solve_outside_the_randomized_regime_is_a_config_error(tmp_path):
    small = str(tmp_path / "small")
    assert run(["gen", "--m", "2", "--n", "6", "--seed", "3", "--out", small])[0] == 0
    assert run(["solve", small + "_A.mtx", small + "_b.mtx"])[0] == 4  # default l = 8 >= n = 6


@pytest.mark.gpu
def test_bench_csv_and_seed_determinism():
    args = ["bench", "--grid", "4:64:16,4:8:16", "--trials", "2", "--kappa", "1e3", "--seed", "21"]
    rc1, csv1, err = run(args)
    rc2, csv2, _ = run(args)
    assert rc1 == 4 and rc2 == 4 and "failed" in err  # the second grid row is invalid
    assert csv1.startswith("m,n,l,t0,tr,ratio,eps0,epsr\n") and "4,64,16," in csv1
    assert csv1.strip().split(",")[-1] == csv2.strip().split(",")[-1]  # error columns are deterministic
    assert run(["bench", "--grid", "4:64:16", "--trials", "1", "--kappa", "1", "--seed", "22"])[0] == 0


@pytest.mark.gpu
def test_selftest_passes_and_the_fault_hook_is_caught():
    rc, out, _ = run(["selftest"])
    assert rc == 0 and "FAIL" not in out and out.strip().endswith("passed")
    rc, out, _ = run(["selftest", "--corrupt-dft"])
    assert rc == 1 and "FAIL srft / dft matches the direct formula" in out
