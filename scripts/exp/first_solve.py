#!/usr/bin/env python
"""Diagnostic: the first solve in a fresh context at a BASELINE config, host vs device x."""
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
    cfg = bench.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A = bench.make_A_shard(cfg, 0, cfg["n"], dev)
    b = bench.make_b(cfg)
    free, total = torch.cuda.mem_get_info()
    print(f"{name}: torch allocated {torch.cuda.memory_allocated() / 2**30:.1f} GiB, reserved "
          f"{torch.cuda.memory_reserved() / 2**30:.1f} GiB, free {free / 2**30:.1f} GiB", flush=True)
    scfg = mn.SolverConfig(epsilon=cfg["eps"], seed=42)
    xs = []
    for mode in ("host", "host", "device"):
        ctx = mn.Context(0)
        ctx.set_matrix(A)
        xd = torch.empty(cfg["n"], dtype=torch.complex128, device=dev) if mode == "device" else None
        rep = mn.solve_randomized(mn.ProblemInstance(None, b), scfg, ctx, x_out=xd)
        x = xd.cpu().numpy() if xd is not None else rep.x
        rep2 = mn.solve_randomized(mn.ProblemInstance(None, b), scfg, ctx, x_out=xd)
        x2 = xd.cpu().numpy() if xd is not None else rep2.x
        print(mode, "first:", rep.lsq_converged, rep.lsq_iterations, [round(v, 1) for v in rep.extra["sketch_kernel_ms"]],
              "second:", rep2.lsq_converged, rep2.lsq_iterations, [round(v, 1) for v in rep2.extra["sketch_kernel_ms"]],
              "rel first vs second %.3e" % (np.linalg.norm(x - x2) / np.linalg.norm(x2)), flush=True)
        xs.append(x2)
        ctx.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
