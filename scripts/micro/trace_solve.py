import sys; sys.path.insert(0,'/root/repo')
import torch, bench, paper_0905_4745_b200 as mn
cfg = bench.CONFIGS[sys.argv[1]]
dev = torch.device("cuda", 0)
ctx = mn.Context(0); ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
A = bench.make_A_shard(cfg, 0, cfg["n"], dev); b = bench.make_b(cfg)
ctx.set_matrix(A, n_global=cfg["n"])
x = torch.empty(cfg["n"], dtype=torch.complex128, device=dev)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    print("---- solve", i, file=sys.stderr, flush=True)
    mn.solve_randomized(mn.ProblemInstance(None, b), mn.SolverConfig(epsilon=cfg["eps"]), ctx, x_out=x)
