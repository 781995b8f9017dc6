"""Micro-benchmark of the SRFT sketch T·A^H alone on a device-resident A:
python scripts/bench_sketch.py [m n real reps] -- prints per-call ms."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0905_4745_b200 as mn

m, n, real, reps = 2048, 1 << 20, 0, 3
if len(sys.argv) > 1:
    m, n, real, reps = (int(x) for x in sys.argv[1:5])
ctx = mn.Context(0)
dt = torch.float64 if real else torch.complex128
At = torch.randn((n, m), dtype=dt, device="cuda")
ctx.set_matrix(At.T, n_global=n)
op = mn.build_srft(4 * m, n, stream_seed=mn.derive_seed(42, 11))
out = torch.empty((m, 4 * m), dtype=torch.complex128, device="cuda")  # l x m column-major
import ctypes
from paper_0905_4745_b200 import _lib as L
lib = L.load()
def run():
    st = lib.mnb_srft_apply_to_columns(ctx._h, op._h, ctypes.c_void_p(out.data_ptr()), L.MNB_DEVICE)
    assert st == 0, L.last_error()
run()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(reps):
    run()
torch.cuda.synchronize()
print(json.dumps({"m": m, "n": n, "real": real, "ms_per_sketch": (time.perf_counter() - t) / reps * 1e3}))
