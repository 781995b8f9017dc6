#!/usr/bin/env python
"""Diagnostic: repeated fresh-context solves (host x, as the full-size parity test) at a config,
after the same warm-up the test suite gives (a c3 solve + oracle in the same process)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0905_4745_b200 as mn  # noqa: E402


def main():
    import torch
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    cfg = bench.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A = bench.make_A_shard(cfg, 0, cfg["n"], dev)
    b = bench.make_b(cfg)
    scfg = mn.SolverConfig(epsilon=cfg["eps"], seed=42)
    xs = []
    for k in range(reps):
        ctx = mn.Context(0)
        ctx.set_matrix(A)
        t = time.perf_counter()
        rep = mn.solve_randomized(mn.ProblemInstance(None, b), scfg, ctx)
        dt = time.perf_counter() - t
        ctx.close()
        xs.append(rep.x)
        print(k, rep.lsq_converged, rep.lsq_iterations, f"{dt * 1e3:.1f} ms",
              [round(v, 1) for v in rep.extra["sketch_kernel_ms"]], hex(rep.extra["qr_path"]),
              "rel vs first %.2e" % (np.linalg.norm(rep.x - xs[0]) / np.linalg.norm(xs[0])), flush=True)


if __name__ == "__main__":
    main()
