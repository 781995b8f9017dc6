#!/usr/bin/env python
"""Diagnostic: the c4 solve with the sketch forced into row slabs of various heights
(MNB_SLAB_ROWS), against the single-slab solve: convergence, iterations, x difference, and the
sketch itself (apply_to_columns of T on the same A)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0905_4745_b200 as mn  # noqa: E402


def main():
    import torch
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    sizes = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "0,1024,1000,600,592,296,1184").split(",")]
    cfg = bench.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A = bench.make_A_shard(cfg, 0, cfg["n"], dev)
    b = bench.make_b(cfg)
    scfg = mn.SolverConfig(epsilon=cfg["eps"], seed=42)
    op = mn.build_srft(4 * cfg["m"], cfg["n"], mn.derive_seed(42, 11))
    ref_x = ref_S = None
    for rows in sizes:
        if rows:
            os.environ["MNB_SLAB_ROWS"] = str(rows)
        else:
            os.environ.pop("MNB_SLAB_ROWS", None)
        ctx = mn.Context(0)
        ctx.set_matrix(A)
        rep = mn.solve_randomized(mn.ProblemInstance(None, b), scfg, ctx)
        S = op.sketch(ctx)
        ctx.close()
        if ref_x is None:
            ref_x, ref_S = rep.x, S
        dS = np.abs(S - ref_S).max() / np.abs(ref_S).max()
        bad_cols = int(np.sum(np.any(S != ref_S, axis=0)))
        print(f"slab {rows}: converged {rep.lsq_converged} it {rep.lsq_iterations} rel x "
              f"{np.linalg.norm(rep.x - ref_x) / np.linalg.norm(ref_x):.2e} sketch max rel {dS:.2e} "
              f"cols differing {bad_cols} kernel ms {[round(v, 1) for v in rep.extra['sketch_kernel_ms']]}", flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
