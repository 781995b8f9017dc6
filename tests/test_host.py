"""CPU-only tests of the product's host side (no GPU needed):

* libminnorm_b200.so loads and exports every symbol include/minnorm_b200.h declares;
* the host SRFT parameter generator is bit-identical to the reference
  RandomStream (golden vectors from oracle/_ref, the oracle, and SURVEY §8c);
* argument checks mirror the reference (build_srft, src/srft.cpp:97-98);
* the multi-GPU column partition.
"""
import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_0905_4745_b200 as mn
from paper_0905_4745_b200 import _lib
from oracle import minnorm_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    with open(os.path.join(ROOT, "include", "minnorm_b200.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(mnb_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.mnb_version().startswith(b"minnorm_b200")


def test_library_is_sm100a_only():
    """The shipped fatbin carries sm_100a SASS (cuobjdump) and no other arch."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_host_params_match_golden_vectors():
    with open(os.path.join(ROOT, "tests", "golden", "srft_golden.json")) as f:
        g = json.load(f)
    for case in g["operators"]:
        op = mn.build_srft(case["l"], case["n"], case["stream_seed"])
        for name, h in case["sha256"].items():
            assert _sha(op.field(name)) == h, (case["n"], name)


@pytest.mark.parametrize("l,n,seed", [(3, 8, 1), (17, 40, 31), (1, 2, 5), (100, 6144, 77), (4096, 1 << 17, 9), (8192, 1 << 20, 11)])
@pytest.mark.parametrize("without", [True, False])
def test_host_params_bit_identical_to_oracle(l, n, seed, without):
    mode = mn.Sampling.without_replacement if without else mn.Sampling.with_replacement
    op = mn.build_srft(l, n, seed, mode)
    ref = O.Srft.build(l, n, seed, without)
    for name in _lib.FIELDS:
        a, b = op.field(name), ref.field(name)
        assert a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8)), name


def test_survey_golden_values_from_product():
    op = mn.build_srft(8192, 1 << 20, mn.derive_seed(42, 11))
    assert op.field("sample")[:4].tolist() == [413293, 426576, 565453, 361359]
    assert int(op.field("perm")[0]) == 499701
    op = mn.build_srft(16384, 3 << 20, mn.derive_seed(42, 11))
    assert op.field("sample")[:4].tolist() == [413293, 1078125, 784681, 1045796]
    assert int(op.field("perm")[0]) == 1447875


def test_derive_seed_matches_reference_rule():
    for s in (0, 42, 2**64 - 1):
        for t in range(1, 13):
            assert mn.derive_seed(s, t) == O.derive_seed(s, t)


def test_build_rejects_bad_shapes():
    """tests/test_srft.cpp:44-52"""
    for l, n in ((9, 8), (1, 1), (0, 8)):
        with pytest.raises(ValueError):
            mn.build_srft(l, n, 1)


def test_field_counts_and_determinism():
    """tests/test_srft.cpp:15-33"""
    op = mn.build_srft(2, 2, 5)
    assert op.field("theta").size == 1 and op.field("d").size == 2 and op.field("sample").size == 2
    a, b = mn.build_srft(5, 16, 77), mn.build_srft(5, 16, 77)
    for f in _lib.FIELDS:
        assert np.array_equal(a.field(f), b.field(f))


def test_unit_modulus_and_bijection():
    """tests/test_srft.cpp:35-42"""
    op = mn.build_srft(4, 8, 9)
    for f in ("d", "zeta", "zeta_tilde"):
        assert np.all(np.abs(np.abs(op.field(f)) - 1) <= 1e-15)
    assert len(set(op.field("sample").tolist())) == 4
    assert sorted(op.field("perm").tolist()) == list(range(8))


@pytest.mark.parametrize("n,world", [(10, 3), (1 << 20, 8), (7, 8), (3 << 20, 4), (1, 1)])
def test_shard_columns_partition(n, world):
    spans = [mn.shard_columns(n, world, r) for r in range(world)]
    assert spans[0][0] == 0
    for (b0, c0), (b1, _) in zip(spans, spans[1:]):
        assert b0 + c0 == b1
    assert sum(c for _, c in spans) == n
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
