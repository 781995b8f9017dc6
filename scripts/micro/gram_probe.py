"""Gram-matrix (S^H S, S l x m complex128) throughput probes: one GEMM vs K-split batched GEMMs."""
import json, torch
def bench(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
out = {}
for m in (2048, 4096):
    l = 4 * m
    S = torch.randn(l, m, dtype=torch.complex128, device="cuda")
    fl = 8 * l * m * m
    ms = bench(lambda: S.mH @ S); out[f"gemm_{l}x{m}"] = (ms, fl / ms / 1e9)
    for k in (2, 4, 8):
        Sb = S.view(k, l // k, m)
        ms = bench(lambda: torch.bmm(Sb.mH, Sb).sum(0)); out[f"bmm{k}_{l}x{m}"] = (ms, fl / ms / 1e9)
print(json.dumps(out, indent=1))
