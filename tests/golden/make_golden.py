"""Generates tests/golden/*.json from the reference's OWN rng.cpp, compiled
verbatim into oracle/_ref/libminnorm_ref.so (oracle/Makefile target `ref`).

SRFT parameter fields are composed from the reference rng primitives exactly
as build_srft does (src/srft.cpp:95-113, tags :13-22); full arrays are pinned
by SHA-256, heads by value.  Run from the repo root:
    python tests/golden/make_golden.py
"""
import ctypes
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import minnorm_oracle as O  # noqa: E402  (only to build / load oracle/_ref)

O.build()
R = O.ref_lib()
assert R is not None, "oracle/_ref/libminnorm_ref.so missing (needs /root/reference)"
P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731


def u64(seed, n):
    a = np.zeros(n, np.uint64)
    R.ref_rng_u64(seed, n, P(a))
    return a


def draw(seed, kind, n):
    a = np.zeros(n * (2 if kind in (2, 4) else 1))
    R.ref_rng_draw(seed, kind, n, P(a))
    return a


def perm(seed, n):
    a = np.zeros(n, np.int64)
    R.ref_rng_permutation(seed, n, P(a))
    return a


def sample(seed, l, n, without):
    a = np.zeros(l, np.int64)
    assert R.ref_rng_sample(seed, l, n, int(without), P(a)) == 0
    return a


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


streams = []
for seed in [0, 1, 42, 2**63 + 5, 0xFFFFFFFFFFFFFFFF]:
    streams.append({
        "seed": seed,
        "u64": [str(int(v)) for v in u64(seed, 16)],
        "angle": draw(seed, 1, 8).tolist(),
        "unit_circle": draw(seed, 2, 4).tolist(),
        "perm17": perm(seed, 17).tolist(),
        "sample_without": sample(seed, 5, 17, True).tolist(),
        "sample_with": sample(seed, 5, 17, False).tolist(),
        "derive": [int(R.ref_derive_seed(seed, t)) for t in range(1, 13)],
    })
with open(os.path.join(ROOT, "tests", "golden", "rng_golden.json"), "w") as f:
    json.dump({"source": "reference src/rng.cpp compiled verbatim (oracle/_ref)", "streams": streams}, f, indent=1)

ops = []
for (l, n, root_seed, tag) in [(256, 1024, 42, 11), (1024, 16384, 42, 12), (4096, 1 << 17, 42, 11),
                               (8192, 1 << 20, 42, 11), (16384, 3 << 20, 42, 12), (3, 8, 7, 11)]:
    s = int(R.ref_derive_seed(root_seed, tag))
    sub = lambda t: int(R.ref_derive_seed(s, t))  # noqa: E731
    fields = {
        "d": draw(sub(1), 2, n),
        "sample": sample(sub(2), l, n, True),
        "theta": draw(sub(3), 1, n - 1),
        "theta_tilde": draw(sub(4), 1, n - 1),
        "perm": perm(sub(5), n),
        "perm_tilde": perm(sub(6), n),
        "zeta": draw(sub(7), 2, n),
        "zeta_tilde": draw(sub(8), 2, n),
    }
    ops.append({"l": l, "n": n, "root_seed": root_seed, "tag": tag, "stream_seed": s,
                "sha256": {k: sha(v) for k, v in fields.items()},
                "sample_head": fields["sample"][:4].tolist(), "perm0": int(fields["perm"][0])})
with open(os.path.join(ROOT, "tests", "golden", "srft_golden.json"), "w") as f:
    json.dump({"source": "reference rng primitives composed as src/srft.cpp:95-113", "operators": ops}, f, indent=1)
print("wrote", len(streams), "streams and", len(ops), "operators")
