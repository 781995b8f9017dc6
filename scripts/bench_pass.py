"""Micro-benchmark of the fused PCG pass s = A(A^H w) alone (CUDA events,
mean over reps) for quick kernel iteration: python scripts/bench_pass.py [m n real]..."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0905_4745_b200 as mn

shapes = [(2048, 1 << 20, 0), (1024, 1 << 17, 0), (256, 1 << 14, 0), (64, 1024, 0), (4096, 3 << 20, 1)]
if len(sys.argv) > 1:
    a = [int(x) for x in sys.argv[1:]]
    shapes = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6554.9
ctx = mn.Context(0)
for m, n, real in shapes:
    dt = torch.float64 if real else torch.complex128
    try:
        At = torch.randn((n, m), dtype=dt, device="cuda")
    except torch.OutOfMemoryError:
        print(json.dumps({"m": m, "n": n, "real": real, "skipped": "oom"})); continue
    ctx.set_matrix(At.T, n_global=n)
    ms = ctx.bench_pcg_pass(20)
    esz = 8 if real else 16
    gbs = esz * m * n / (ms * 1e-3) / 1e9
    print(json.dumps({"m": m, "n": n, "real": real, "ms": ms, "GBps": gbs, "frac": gbs / peak}))
    del At
    ctx._keep = None
    torch.cuda.empty_cache()
