#!/usr/bin/env python
"""Timed CPU baseline: complete solve_randomized runs of the oracle port (the reference's
algorithm restated in oracle/; the reference itself needs Eigen) on the BASELINE instances,
per step like src/solver.cpp:79-120, at 1 host thread (the reference is serial)
and at all host threads (the sketch's column loop may run in parallel).  Nothing
is sampled or scaled: every number is one whole solve.  Writes/merges
profiles/r02/cpu_baseline.json (read by bench.py for its 1-thread figure).

usage: python scripts/cpu_baseline.py [--configs c1,c2,c3,c4] [--threads 1,all] [--out FILE]
Test infrastructure: it imports oracle/ and is never the product.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--threads", default="1,all")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "cpu_baseline.json"))
    args = ap.parse_args()
    import bench

    res = {}
    if os.path.exists(args.out):
        with open(args.out) as f:
            res = json.load(f)
    cores = os.cpu_count() or 1
    for name in args.configs.split(","):
        cfg = bench.CONFIGS[name]
        t = time.perf_counter()
        A, b = bench.host_instance(cfg)
        gen = time.perf_counter() - t
        rec = res.get(name, {})
        rec.update({"m": cfg["m"], "n": cfg["n"], "kappa": cfg["kappa"], "epsilon": cfg["eps"],
                    "host": {"cores": cores, "cpu": platform.processor() or platform.machine()},
                    "gen_seconds": gen})
        for th in args.threads.split(","):
            threads = cores if th == "all" else int(th)
            dt, ref = bench.cpu_solve(cfg, A, b, threads)
            rec[f"threads_{'all' if th == 'all' else threads}"] = {
                "threads": threads, "seconds": dt, "step_seconds": [float(s) for s in ref.step_seconds],
                "lsq_iterations": ref.lsq_iterations, "lsq_converged": ref.lsq_converged,
                "residual_norm": ref.residual_norm}
            print(f"{name} threads={threads}: {dt:.2f} s, {ref.lsq_iterations} iterations, "
                  f"steps {[round(s, 3) for s in ref.step_seconds]}", flush=True)
            res[name] = rec
            os.makedirs(os.path.dirname(args.out), exist_ok=True)
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1)
        del A


if __name__ == "__main__":
    main()
