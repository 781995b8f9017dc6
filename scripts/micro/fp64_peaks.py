"""FP64 throughput probes on the GPU (torch -> cuBLAS/cuSOLVER): complex GEMM,
HERK-shaped product, QR, Cholesky at the sketch-QR shapes (l = 4m)."""
import json, time, torch
dev = "cuda"
def bench(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
out = {}
for dt, name in [(torch.float64, "f64"), (torch.complex128, "c128")]:
    a = torch.randn(8192, 8192, dtype=dt, device=dev); b = torch.randn(8192, 8192, dtype=dt, device=dev)
    ms = bench(lambda: a @ b)
    fl = 2 * 8192**3 * (4 if dt == torch.complex128 else 1)
    out[f"gemm_{name}_8192_TFs"] = fl / ms / 1e9
for m in (1024, 2048, 4096):
    l = 4 * m
    S = torch.randn(l, m, dtype=torch.complex128, device=dev)
    ms = bench(lambda: S.mH @ S, 3)
    out[f"gram_c128_{l}x{m}_ms"] = ms
    ms = bench(lambda: torch.linalg.qr(S, mode="r"), 2)
    out[f"qr_r_c128_{l}x{m}_ms"] = ms
    G = S.mH @ S
    ms = bench(lambda: torch.linalg.cholesky(G), 3)
    out[f"chol_c128_{m}_ms"] = ms
    R = torch.linalg.cholesky(G).mH
    ms = bench(lambda: torch.linalg.solve_triangular(R, S, upper=True, left=False), 3)
    out[f"trsm_c128_{l}x{m}_ms"] = ms
print(json.dumps(out, indent=1))
