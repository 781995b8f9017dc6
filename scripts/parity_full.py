#!/usr/bin/env python
"""Full-size parity campaign: the GPU solve against the CPU oracle on the
BASELINE.json configs at their full sizes (c5 on a same-n analog), written to
one JSON file (profiles/r02/parity.json).

Per config:
  * A, b from bench.py's generator (A built on the GPU, the same bits copied
    to the host for the oracle);
  * the GPU randomized solve (A resident, the default paths) and the GPU
    classical solve;
  * the oracle's solve_randomized (oracle/minnorm_oracle.py, the reference's
    algorithm restated; all host threads) -- its x, iteration count and
    per-step wall times (src/solver.cpp:79-120 semantics);
  * the exact minimal-norm p: extended-precision refinement (exact_minnorm)
    where it converges (kappa <= 1e6: c1, c2, c4, c5a), the pivoted-QR
    classical oracle (solve_classical, src/solver.cpp:130-146) elsewhere and
    as the backward-stable yardstick where it fits in host time;
  * relative differences, the conditioning floor u*kappa and 10*eps.

usage: python scripts/parity_full.py [--configs c1,c2,c3,c4,c5a] [--out FILE]
       [--threads N] [--slab-rows R]
This is test infrastructure (it imports oracle/); nothing here is timed as the
product.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ANALOGS = {
    # c5 on a same-n analog: n = 3*2^20 real (the mixed-radix path), kappa and eps of c5, m = 512
    "c5a": dict(m=512, n=3 << 20, kappa=1e6, eps=1e-10, real=True),
    # the same at m = 256, n = 3*2^18 (the analog tests/test_gpu_parity_full.py asserts on)
    "c5s": dict(m=256, n=3 << 18, kappa=1e6, eps=1e-10, real=True),
    # c5's shape with the multi-slab sketch path forced (MNB_SLAB_ROWS): same instance as c5a
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c5s,c4,c5a")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "parity.json"))
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--no-exact", action="store_true")
    args = ap.parse_args()

    import numpy as np
    import torch

    import bench
    import paper_0905_4745_b200 as mn
    from oracle import minnorm_oracle as O

    u = float(np.finfo(np.float64).eps)
    dev = torch.device("cuda", 0)
    results = {}
    if os.path.exists(args.out):
        with open(args.out) as f:
            results = json.load(f)

    def rel(x, y):
        return float(np.linalg.norm(x - y) / np.linalg.norm(y))

    for name in args.configs.split(","):
        cfg = dict(bench.CONFIGS.get(name) or ANALOGS[name])
        m, n, kappa, eps, real = cfg["m"], cfg["n"], cfg["kappa"], cfg["eps"], cfg["real"]
        rec = {"m": m, "n": n, "kappa": kappa, "epsilon": eps, "real": real, "u_kappa": u * kappa,
               "ten_eps": 10 * eps, "host_threads": args.threads}
        print(f"== {name}: m={m} n={n} kappa={kappa:g} eps={eps:g} real={real}", flush=True)
        t0 = time.perf_counter()
        A = bench.make_A_shard(cfg, 0, n, dev)
        b = bench.make_b(cfg)
        torch.cuda.synchronize()
        rec["gen_seconds"] = time.perf_counter() - t0
        scfg = mn.SolverConfig(epsilon=eps, seed=42)
        inst = mn.ProblemInstance(None, b)

        # ---- GPU randomized (default paths; then the multi-slab sketch path for the c5 analog)
        def gpu_solve(env=None):
            old = {}
            for k, v in (env or {}).items():
                old[k] = os.environ.get(k)
                os.environ[k] = v
            try:
                ctx = mn.Context(0)
                ctx.set_matrix(A, n_global=n)
                xd = torch.empty(n, dtype=torch.complex128, device=dev)
                mn.solve_randomized(inst, scfg, ctx, x_out=xd)  # warm
                torch.cuda.synchronize()
                t = time.perf_counter()
                rep = mn.solve_randomized(inst, scfg, ctx, x_out=xd)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t
                x = xd.cpu().numpy()
                ctx.close()
                return x, rep, dt
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v

        x_gpu, rep, dt = gpu_solve()
        rec["gpu"] = {"seconds": dt, "lsq_iterations": rep.lsq_iterations, "lsq_converged": rep.lsq_converged,
                      "residual_norm": rep.residual_norm, "c_norm_ratio": rep.c_norm_ratio,
                      "qr_path": rep.extra["qr_path"], "achieved_excess": rep.extra["lsq_achieved_excess"]}
        print(f"   gpu: {dt*1e3:.1f} ms, it {rep.lsq_iterations}, qr_path {rep.extra['qr_path']:#x}", flush=True)
        if name == "c5a":
            x_slab, rep_slab, dt_slab = gpu_solve({"MNB_SLAB_ROWS": "64"})  # 8 slabs of 64 rows (Ms < m)
            rec["gpu_multislab"] = {"slab_rows": 64, "seconds": dt_slab, "lsq_iterations": rep_slab.lsq_iterations,
                                    "rel_vs_default_slab": rel(x_slab, x_gpu)}
        # ---- GPU classical (the paper's t0 solver on the device)
        ctx = mn.Context(0)
        ctx.set_matrix(A, n_global=n)
        t = time.perf_counter()
        x_cls, crep = mn.solve_classical(inst, ctx, report=True)
        rec["gpu_classical"] = {"seconds": time.perf_counter() - t, "path": crep.path,
                                "refinements": crep.refinements}
        ctx.close()
        # Gram matrix for the exact-p refinement (float64, on the GPU: test infrastructure)
        G = None
        if not args.no_exact and kappa <= 1e6:
            G = (A @ A.conj().T).cpu().numpy()
            G = G.astype(np.complex128)
        # ---- host copy of the same bits
        A_host = A.T.contiguous().cpu().numpy().T  # m x n, column-major
        del A
        torch.cuda.empty_cache()
        # ---- oracle randomized solve (the reference's algorithm)
        t = time.perf_counter()
        ref = O.solve_randomized(A_host, b, epsilon=eps, seed=42, threads=args.threads)
        rec["oracle"] = {"seconds": time.perf_counter() - t, "step_seconds": ref.step_seconds,
                         "lsq_iterations": ref.lsq_iterations, "lsq_converged": ref.lsq_converged,
                         "residual_norm": ref.residual_norm, "c_norm_ratio": ref.c_norm_ratio}
        print(f"   oracle: {rec['oracle']['seconds']:.1f} s, it {ref.lsq_iterations}, conv {ref.lsq_converged}",
              flush=True)
        if not ref.lsq_converged and name != "c5a":
            # the reference given the GPU's iteration budget (its own SolverConfig.lsq_max_iterations knob)
            ref_k = O.solve_randomized(A_host, b, epsilon=eps, seed=42, threads=args.threads,
                                       lsq_max_iterations=rep.lsq_iterations)
        else:
            ref_k = None
        rec["rel_gpu_vs_oracle"] = rel(x_gpu, ref.x)
        rec["iterations_gpu_minus_oracle"] = rep.lsq_iterations - ref.lsq_iterations
        rec["rel_gpu_vs_gpu_classical"] = rel(x_gpu, x_cls)
        # ---- exact p
        p = None
        if G is not None:
            t = time.perf_counter()
            p, hist = O.exact_minnorm(A_host, b, G=G)
            rec["exact"] = {"method": "extended-precision y-space refinement (oracle.exact_minnorm)",
                            "seconds": time.perf_counter() - t, "residual_history": hist}
        qr_ok = m * n <= (1 << 27) or (real and m <= 512)
        if qr_ok:
            t = time.perf_counter()
            p_qr = O.solve_classical(A_host, b)
            rec["pivoted_qr_seconds"] = time.perf_counter() - t
            if p is None:
                p = p_qr
                rec["exact"] = {"method": "pivoted Householder QR (oracle.solve_classical; floor ~u*kappa)"}
            else:
                rec["rel_pivoted_qr_vs_p"] = rel(p_qr, p)
        if p is not None:
            rec["rel_gpu_vs_p"] = rel(x_gpu, p)
            rec["rel_oracle_vs_p"] = rel(ref.x, p)
            rec["rel_gpu_classical_vs_p"] = rel(x_cls, p)
            if ref_k is not None:
                rec["rel_oracle_at_gpu_iterations_vs_p"] = rel(ref_k.x, p)
                rec["rel_gpu_vs_oracle_at_gpu_iterations"] = rel(x_gpu, ref_k.x)
            if name == "c5a":
                rec["gpu_multislab"]["rel_vs_p"] = rel(x_slab, p)
        rec["true_residual_gpu"] = float(np.linalg.norm(O.A_r(A_host, x_gpu) - b))
        results[name] = rec
        print("   " + json.dumps({k: v for k, v in rec.items() if k.startswith("rel") or k.startswith("iter")}),
              flush=True)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(results, f, indent=1)
        del A_host, G, p
    print("done")


if __name__ == "__main__":
    main()
