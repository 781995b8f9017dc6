import sys, os, json, subprocess, threading, time
sys.path.insert(0, '/root/repo')
import torch, paper_0905_4745_b200 as mn
ctx = mn.Context(0)
m, n = 2048, 1 << 20
At = torch.randn((n, m), dtype=torch.complex128, device="cuda")
ctx.set_matrix(At.T, n_global=n)
for reps in (10, 50, 200):
    ms = ctx.bench_pcg_pass(reps)
    print(json.dumps({"reps": reps, "ms": ms, "GBps": 16 * m * n / ms / 1e6}))
