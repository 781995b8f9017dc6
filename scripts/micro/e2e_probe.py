"""e2e probe at c4: host (pinned) A through solve_randomized, with the report's step breakdown."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench, paper_0905_4745_b200 as mn
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
dev = torch.device("cuda", 0)
ctx = mn.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
A = bench.make_A_shard(cfg, 0, cfg["n"], dev)
b = bench.make_b(cfg)
A_host = torch.empty((cfg["n"], cfg["m"]), dtype=A.dtype, pin_memory=True)
A_host.copy_(A.T)
del A
torch.cuda.empty_cache()
A_np = A_host.numpy().T
scfg = mn.SolverConfig(epsilon=cfg["eps"], seed=42)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = mn.solve_randomized(mn.ProblemInstance(A_np, b), scfg, ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    e = rep.extra
    print(json.dumps({"e2e_s": dt, "steps": rep.step_seconds, "param": e["param_seconds"], "total_host": e["total_seconds"],
                      "sketch": e["sketch_seconds"], "qr": e["qr_seconds"], "pcg": e["pcg_seconds"], "iters": rep.lsq_iterations}))
