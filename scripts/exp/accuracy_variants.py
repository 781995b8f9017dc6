#!/usr/bin/env python
"""Diagnostic (test infrastructure): where does the randomized GPU solve lose accuracy against the
exact p at the kappa = 1e6 configs?  Runs GPU solves under the solver's env switches on the bench
instance and reports ||x - p|| / ||p||, p from the oracle's pivoted QR (solve_classical)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0905_4745_b200 as mn  # noqa: E402
from oracle import minnorm_oracle as O  # noqa: E402

VARIANTS = {"default": {}, "csne0": {"MNB_CSNE": "0"}, "householder": {"MNB_QR": "householder"},
            "init_pass": {"MNB_INIT_PASS": "1"}, "no2norm": {"MNB_PRECOND_2NORM": "0"},
            "csne0_init_pass": {"MNB_CSNE": "0", "MNB_INIT_PASS": "1"}}


def main():
    import torch
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cfg = dict(bench.CONFIGS.get(name) or dict(m=256, n=3 << 18, kappa=1e6, eps=1e-10, real=True))
    dev = torch.device("cuda", 0)
    A = bench.make_A_shard(cfg, 0, cfg["n"], dev)
    b = bench.make_b(cfg)
    Ah = A.T.cpu().numpy().T
    p = O.solve_classical(Ah, b)
    out = {}
    for vn, env in VARIANTS.items():
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            ctx = mn.Context(0)
            ctx.set_matrix(A)
            rep = mn.solve_randomized(mn.ProblemInstance(None, b), mn.SolverConfig(epsilon=cfg["eps"]), ctx)
            x = rep.x
            ctx.close()
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        out[vn] = {"rel_vs_p": float(np.linalg.norm(x - p) / np.linalg.norm(p)), "it": rep.lsq_iterations,
                   "qr_path": hex(rep.extra["qr_path"]), "ms": rep.extra["total_seconds"] * 1e3}
        print(name, vn, json.dumps(out[vn]), flush=True)
    for it in (rep.lsq_iterations,):
        r = O.solve_randomized(Ah, b, epsilon=cfg["eps"], lsq_max_iterations=it, threads=os.cpu_count())
        print(name, f"oracle@{it}", float(np.linalg.norm(r.x - p) / np.linalg.norm(p)), flush=True)


if __name__ == "__main__":
    main()
