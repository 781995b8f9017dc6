"""Kernel times of the hand-written Cholesky / triangular inverse (k_cholqr.cu) beside the
library routines they replaced (cuSOLVER potrf, a triangular solve against I; through torch),
on Gram matrices of BASELINE-shaped sketches.  Run on a GPU box: python scripts/bench_cholqr.py"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0905_4745_b200 as mn  # noqa: E402


def main():
    ctx = mn.Context(0)
    rows = []
    for m in (64, 256, 1024, 2048, 4096):
        l = 4 * m
        g = torch.Generator(device="cuda").manual_seed(m)
        S = torch.randn(l, m, dtype=torch.complex128, device="cuda", generator=g)
        S = S * torch.logspace(0, -3, m, dtype=torch.float64, device="cuda")
        G = (S.mH @ S)
        Gh = G.cpu().numpy()
        ours = []
        for _ in range(4):
            R, st = ctx.chol_upper(Gh)
            ours.append(st["kernel_ms"])
        inv = []
        for _ in range(4):
            X, _ = ctx.trtri_upper(R)
            inv.append(ctx.last_kernel_ms)
        # library: potrf and a triangular solve against the identity
        lib_c, lib_i = [], []
        eye = torch.eye(m, dtype=torch.complex128, device="cuda")
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Rl = torch.linalg.cholesky(G, upper=True)
            torch.cuda.synchronize()
            lib_c.append((time.perf_counter() - t0) * 1e3)
            t0 = time.perf_counter()
            Xl = torch.linalg.solve_triangular(Rl, eye, upper=True)
            torch.cuda.synchronize()
            lib_i.append((time.perf_counter() - t0) * 1e3)
        err = float(np.linalg.norm(R - Rl.cpu().numpy()) / np.linalg.norm(R))
        rows.append({"m": m, "chol_ms": min(ours), "trtri_ms": min(inv), "potrf_lib_ms": min(lib_c),
                     "trsm_identity_lib_ms": min(lib_i), "rel_diff_R": err})
        print(rows[-1], flush=True)
    json.dump(rows, open("gpurun_out/bench_cholqr.json", "w"), indent=1)


if __name__ == "__main__":
    main()
