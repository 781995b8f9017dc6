"""Step-time jitter of back-to-back solves with and without an in-process NVML
sampler thread; also times each NVML query.  python scripts/micro/jitter_probe.py c3 30"""
import sys, time, threading, statistics, resource
sys.path.insert(0, '/root/repo')
import torch, bench, paper_0905_4745_b200 as mn
import pynvml

cfg = bench.CONFIGS[sys.argv[1]]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
dev = torch.device("cuda", 0)
ctx = mn.Context(0); ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
A = bench.make_A_shard(cfg, 0, cfg["n"], dev); b = bench.make_b(cfg)
ctx.set_matrix(A, n_global=cfg["n"])
x = torch.empty(cfg["n"], dtype=torch.complex128, device=dev)
inst = mn.ProblemInstance(None, b); scfg = mn.SolverConfig(epsilon=cfg["eps"])
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
qt = {"clock": [], "reasons": []}

def run(mode):
    stop = threading.Event()
    def sampler():
        while not stop.is_set():
            t = time.perf_counter(); pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); qt["clock"].append(time.perf_counter() - t)
            if mode == "full":
                t = time.perf_counter(); pynvml.nvmlDeviceGetCurrentClocksEventReasons(h); qt["reasons"].append(time.perf_counter() - t)
            stop.wait(0.1)
    th = threading.Thread(target=sampler, daemon=True)
    if mode != "none": th.start()
    st = torch.cuda.current_stream(dev)
    ms = []; flt = []; reps = []
    for _ in range(steps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        r0 = resource.getrusage(resource.RUSAGE_SELF)
        e0.record(st); rep = mn.solve_randomized(inst, scfg, ctx, x_out=x); e1.record(st); e1.synchronize()
        reps.append(rep)
        r1 = resource.getrusage(resource.RUSAGE_SELF)
        ms.append(e0.elapsed_time(e1))
        flt.append((r1.ru_minflt - r0.ru_minflt, r1.ru_majflt - r0.ru_majflt, r1.ru_nivcsw - r0.ru_nivcsw, r1.ru_nvcsw - r0.ru_nvcsw))
    stop.set()
    if mode != "none": th.join()
    med = statistics.median(ms)
    print(f"{mode:6s} median {med:8.2f} ms  max {max(ms):8.2f}  outliers(>1.2x) {[round(v,1) for v in ms if v > 1.2*med]}", flush=True)
    print("   (minflt, majflt, nivcsw, nvcsw) normal:", [f for v, f in zip(ms, flt) if v <= 1.2 * med][:6], flush=True)
    def brk(r):
        e = r.extra
        return dict(sk=[round(v * 1e3, 1) for v in e["sketch_seconds"]], qr=[round(v * 1e3, 1) for v in e["qr_seconds"]],
                    pcg=round(e["pcg_seconds"] * 1e3, 1), par=round(e["param_seconds"] * 1e3, 1),
                    st=[round(v * 1e3, 1) for v in r.step_seconds])
    print("   normal breakdown:", [brk(r) for v, r in zip(ms, reps) if v <= 1.2 * med][:2], flush=True)
    print("   outlier breakdown:", [(round(v, 1), brk(r)) for v, r in zip(ms, reps) if v > 1.2 * med][:6], flush=True)
    print("   outliers:", [(round(v, 1),) + f for v, f in zip(ms, flt) if v > 1.2 * med][:12], flush=True)

for _ in range(3): mn.solve_randomized(inst, scfg, ctx, x_out=x)
for mode in ("none", "clock", "full", "none", "full"):
    run(mode)
for k, v in qt.items():
    if v: print(k, "query ms: median %.3f max %.3f" % (1e3*statistics.median(v), 1e3*max(v)))
