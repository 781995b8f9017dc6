#!/usr/bin/env python
"""Benchmark of the B200-native randomized minimal-norm solve (arXiv 0905.4745).

One "step" = one full solve_randomized (Steps 1-5, both SRFT sketches, both
QRs, the preconditioned CG, x = A^H y) on one synthetic instance of a
BASELINE.json config (default c4: m=2048, n=2^20 complex128, the
bandwidth-bound PCG regime; A = 32 GiB > the 126 MB L2, so no flush is
needed between steps).  Prints ONE JSON line (rank 0).

  python bench.py [--config c4] [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU: launched with torch.distributed.run, one rank per GPU; A is
column-sharded (strong scaling of one solve), NCCL inside the library.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # BASELINE.json "configs"
    "c1": dict(m=64, n=1024, kappa=1e3, eps=1e-12, real=False),
    "c2": dict(m=256, n=16384, kappa=1e6, eps=1e-10, real=False),
    "c3": dict(m=1024, n=131072, kappa=1e8, eps=1e-10, real=False),
    "c4": dict(m=2048, n=1 << 20, kappa=1e4, eps=1e-8, real=False),
    "c5": dict(m=4096, n=3 << 20, kappa=1e6, eps=1e-10, real=True),
}
METRIC = "min-norm solve time; HBM GB/s of fused PCG A(A*y) pass & SRFT sketch vs peak"
DATA_SEED = 20260101


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_peak_tfs():
    """Measured FP64 peak (DGEMM 8192^3 on this pool's B200, scripts/micro/fp64_peaks.py ->
    profiles/r02/fp64_peaks.json); MEASURED_PEAKS.json has no FP64 figure.  Fallback: 37 TF nominal."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "fp64_peaks.json")) as f:
            return float(json.load(f)["gemm_f64_8192_TFs"]), "measured (DGEMM, profiles/r02/fp64_peaks.json)"
    except Exception:
        return 37.0, "nominal"


# ------------------------------------------------------------------ data ---
def make_A_shard(cfg, col_begin, n_local, device):
    """A[:, col_begin:col_begin+n_local] of A = U diag(sigma) G / sqrt(n), built on
    the GPU chunk by chunk with seeds tied to global column chunks (so every
    world size sees the same bits).  Column-major (returned as A with strides (1, m))."""
    import torch
    m, n, real = cfg["m"], cfg["n"], cfg["real"]
    ctype = torch.float64 if real else torch.complex128
    gU = torch.Generator(device=device).manual_seed(DATA_SEED)
    if real:
        Z = torch.randn((m, m), dtype=torch.float64, device=device, generator=gU)
    else:
        Z = torch.randn((m, m), dtype=torch.complex128, device=device, generator=gU)
    Q, R = torch.linalg.qr(Z)
    d = torch.diagonal(R)
    U = Q * (d / d.abs())
    sigma = torch.logspace(0, -math.log10(cfg["kappa"]), m, dtype=torch.float64, device=device)
    Us = (U * sigma.to(ctype)) / math.sqrt(n)
    At = torch.empty((n_local, m), dtype=ctype, device=device)  # row-major (n x m) == column-major A
    chunk = 1 << 16
    first, last = col_begin // chunk, (col_begin + n_local - 1) // chunk
    for ci in range(first, last + 1):
        g = torch.Generator(device=device).manual_seed(DATA_SEED + 1 + ci)
        c0 = ci * chunk
        width = min(chunk, n - c0)
        G = torch.randn((m, width), dtype=ctype, device=device, generator=g)
        blk = (Us @ G).T  # width x m
        lo, hi = max(c0, col_begin), min(c0 + width, col_begin + n_local)
        At[lo - col_begin:hi - col_begin] = blk[lo - c0:hi - c0]
        del G, blk
    del Z, Q, R, U
    return At.T  # m x n_local, column-major view


def make_b(cfg):
    import numpy as np
    rng = np.random.default_rng(DATA_SEED + 7)
    m = cfg["m"]
    if cfg["real"]:
        return rng.standard_normal(m).astype(np.complex128)
    return (rng.standard_normal(m) + 1j * rng.standard_normal(m)) / np.sqrt(2)


# ---------------------------------------------------------------- clocks ---
class ClockSampler:
    """SM clock / throttle-reason samples during the timed region.  In-process
    NVML polling (a light driver query every 100 ms; spawning nvidia-smi inside
    the timed region stalls millisecond-scale solves); nvidia-smi as fallback."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, device_index: int):
        import threading
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self.stop_flag = threading.Event()
        self.thread = None
        self.proc = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while True:
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, name in self.REASONS.items():
                            if bits & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    if self.stop_flag.wait(0.1):
                        return

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self._start_smi(device_index)

    def _start_smi(self, device_index):
        self.path = tempfile.mktemp(suffix=".csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(device_index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join(timeout=5)
        elif self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=10)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            with open(self.path) as f:
                for line in f:
                    p = [x.strip() for x in line.split(",")]
                    if len(p) < 8:
                        continue
                    try:
                        self.sm.append(float(p[0]))
                        self.mx = max(self.mx, float(p[1]))
                    except ValueError:
                        continue
                    for nm, v in zip(names, p[4:8]):
                        if v.lower() == "active":
                            self.reasons.add(nm)
            os.unlink(self.path)
        if not self.sm:
            return None
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


# ----------------------------------------------------------- CPU baseline --
def host_instance(cfg):
    """(A, b) on the host: A is m x n column-major with the bits make_A_shard builds (on the GPU
    when one is visible, as in the device arm; on the CPU generator otherwise)."""
    import torch
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    A = make_A_shard(cfg, 0, cfg["n"], dev)
    A_host = A.T.cpu().numpy().T  # (n, m) row-major == m x n column-major
    del A
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    return A_host, make_b(cfg)


def cpu_solve(cfg, A_host, b, threads):
    """One COMPLETE solve_randomized of the oracle port (oracle/minnorm_oracle.py: the reference's
    src/solver.cpp:50-128 and src/lsq.cpp:43-113 restated; the reference itself needs Eigen, which
    this image lacks) on this very instance, timed with a wall clock around the call as
    src/solver.cpp:79-120 times its steps.  `threads` bounds both the sketch's column loop
     and OpenBLAS (GEMVs, LAPACK QR).  Returns (seconds, oracle SolveReport)."""
    from threadpoolctl import threadpool_limits

    from oracle import minnorm_oracle as O
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        ref = O.solve_randomized(A_host, b, epsilon=cfg["eps"], seed=42, threads=threads)
        dt = time.perf_counter() - t0
    return dt, ref


def cpu_threads(cfg):
    """Host threads of the CPU port: all cores, except at c1-sized problems (m n <= 2^20), where
    OpenBLAS's thread pools cost more than the work (c1: 0.014 s on 1 thread, 0.30 s on 8);
    MNB_CPU_THREADS overrides."""
    env = os.environ.get("MNB_CPU_THREADS")
    if env:
        return max(1, int(env))
    return 1 if cfg["m"] * cfg["n"] <= (1 << 20) else (os.cpu_count() or 1)


def cpu_record(dt, ref, threads, what):
    return {"value": dt, "unit": "s", "cores": threads, "kind": "port",
            "sample": f"{what}: complete solve_randomized of the oracle port (the reference's algorithm, "
                      f"oracle/minnorm_oracle.py) on this instance, {threads} host threads, not scaled",
            "lsq_iterations": ref.lsq_iterations, "lsq_converged": ref.lsq_converged,
            "step_seconds": [float(s) for s in ref.step_seconds]}


def recorded_single_thread(config_name):
    """The 1-thread figure, measured by scripts/cpu_baseline.py (too long to rerun
    inside every bench call at c3-c5); None when no measurement is committed."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "cpu_baseline.json")) as f:
            rec = json.load(f)[config_name]["threads_1"]
        return {"value": rec["seconds"], "unit": "s", "cores": 1, "kind": "port",
                "lsq_iterations": rec["lsq_iterations"],
                "source": "profiles/r02/cpu_baseline.json (scripts/cpu_baseline.py, complete solve, 1 thread)"}
    except Exception:
        return None


# ----------------------------------------------------------------- main ----
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--classical", action="store_true",
                    help="also time the device classical solve (solve_classical, the paper's t0) on the same A")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` outside torchrun: relaunch as N ranks (one per GPU) on this node
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                  f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:])
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    config_json = {"workload": f"BASELINE {args.config}: m={cfg['m']} n={cfg['n']} "
                               f"{'float64' if cfg['real'] else 'complex128'} kappa={cfg['kappa']:g} "
                               f"eps={cfg['eps']:g} l=4m",
                   "m": cfg["m"], "n": cfg["n"], "l": 4 * cfg["m"], "epsilon": cfg["eps"],
                   "parallelism": f"column-sharded x{world}" if world > 1 else "single GPU",
                   "l2": "A (%.1f GiB) exceeds L2; no flush needed" % (cfg["m"] * cfg["n"] * (8 if cfg["real"] else 16) / 2**30)}

    if args.impl == "reference":
        if rank != 0:
            return
        # Complete solves of the CPU port on the host cores, never a scaled sample.  A c4 solve
        # takes minutes on the host, so the run times as many of the requested W + K solves as
        # fit in MNB_CPU_BUDGET_S (default 180 s; at least one timed solve) and reports exactly
        # what ran: "steps" / "warmup" are the counts performed, "*_requested" the flags.
        A_host, b = host_instance(cfg)
        threads = cpu_threads(cfg)
        budget = float(os.environ.get("MNB_CPU_BUDGET_S", "180"))
        t_begin = time.perf_counter()
        dt, ref = cpu_solve(cfg, A_host, b, threads)
        warm, timed = 0, []
        if dt * (args.warmup + args.steps) <= budget:
            warm = 1  # the first solve was a warm-up
            while warm < args.warmup:
                cpu_solve(cfg, A_host, b, threads)
                warm += 1
        else:
            timed.append(dt)
        while len(timed) < args.steps:
            spent = time.perf_counter() - t_begin
            est = statistics.mean(timed) if timed else dt
            if timed and spent + est > budget:
                break
            dt, ref = cpu_solve(cfg, A_host, b, threads)
            timed.append(dt)
        val = statistics.mean(timed)
        rec = cpu_record(val, ref, threads, f"{len(timed)} timed solve(s) after {warm} warm-up(s)")
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": val, "unit": "s", "n_gpus": world,
            "steps": len(timed), "warmup": warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": val * 1e3, "ms_per_step_all": [t * 1e3 for t in timed],
            "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if cfg["real"] else "c128", "data": "synthetic (seeded)",
            "config": config_json,
            "cpu_baseline": rec,
            "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import numpy as np
    import torch
    import paper_0905_4745_b200 as mn

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        uid = [mn.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = mn.Context.distributed(local, rank, world, uid[0])
    else:
        dist = None
        ctx = mn.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    m, n = cfg["m"], cfg["n"]
    col_begin, n_local = mn.shard_columns(n, world, rank)
    A = make_A_shard(cfg, col_begin, n_local, dev)
    b = make_b(cfg)
    if world > 1:
        ctx.set_shard(A, n_global=n)
    else:
        ctx.set_matrix(A)
    scfg = mn.SolverConfig(epsilon=cfg["eps"], seed=42)
    x_dev = torch.empty(max(n_local, 1), dtype=torch.complex128, device=dev)
    inst = mn.ProblemInstance(None, b)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident arm: A already in HBM
    for _ in range(args.warmup):
        mn.solve_randomized(inst, scfg, ctx, x_out=x_dev)
    barrier()
    clocks = ClockSampler(local)
    reps = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ms = []
    for _ in range(args.steps):
        barrier()
        torch.cuda.nvtx.range_push("solve")  # ncu --nvtx --nvtx-include "solve/" selects the timed solves
        e0.record(stream)
        rep = mn.solve_randomized(inst, scfg, ctx, x_out=x_dev)
        e1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize(dev)
        step_ms.append(max_over_ranks(e0.elapsed_time(e1)))
        reps.append(rep)
    barrier()
    clk = clocks.stop()
    ms = statistics.mean(step_ms)
    value = ms / 1e3
    hbm_peak, peak_kind = peaks()
    esz = 8 if cfg["real"] else 16
    pass_ms = statistics.mean(r.extra["pcg_pass_ms_sum"] / max(1, r.extra["pcg_pass_launches"]) for r in reps)
    pass_bytes = esz * m * n_local + 64 * n_local  # A once + the lagged r / t n-vectors (read + write)
    achieved = pass_bytes / (pass_ms * 1e-3) / 1e9
    traffic = None
    traffic_sketch = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            prof = json.load(f).get(args.config, {})
        traffic = prof.get("pcg_pass_dram_bytes_per_launch")
        traffic_sketch = prof.get("sketch_dram_bytes_per_sketch")
    except Exception:
        pass
    last = reps[-1]
    classical = None
    if args.classical:
        # the paper's comparison t0 / t_r (Tables 1-4) on the GPU: same A (device-resident), same b
        times = []
        for _ in range(2):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            xc, crep = mn.solve_classical(inst, ctx, report=True)
            times.append(time.perf_counter() - t0)
        xr = last.x.cpu().numpy() if hasattr(last.x, "cpu") else np.asarray(last.x)
        classical = {"seconds": min(times), "path": crep.path, "refinements": crep.refinements,
                     "residual_norm": crep.residual_norm,
                     "rel_diff_randomized": float(np.linalg.norm(xr[:n_local] - xc) / np.linalg.norm(xc)),
                     "ratio_t0_over_tr": min(times) / value if value else None,
                     "note": "wall clock of mnb_solve_classical with A in HBM (x to host); value is t_r"}
    sk = last.extra["sketch_kernel_ms"]
    launches = sum(r.extra["kernel_launches"] for r in reps)

    # ---- end-to-end arm: public API with host buffers (H2D of A and b, D2H of x inside the timed region)
    e2e = None
    A_np, rep_h = None, None
    if not args.no_e2e:
        A_host = torch.empty((n_local, m), dtype=A.dtype, pin_memory=True)
        A_host.copy_(A.T)
        A_np = A_host.numpy().T  # m x n_local, column-major view of pinned memory
        del A
        ctx._keep = None
        torch.cuda.empty_cache()
        inst_h = mn.ProblemInstance(A_np, b)
        e2e_ms = []
        for i in range(max(1, args.warmup // 2) + args.steps):
            barrier()
            t0 = time.perf_counter()
            rep_h = mn.solve_randomized(inst_h, scfg, ctx)  # set_matrix(host) + solve + x to host
            torch.cuda.synchronize(dev)
            dt = max_over_ranks((time.perf_counter() - t0) * 1e3)
            if i >= max(1, args.warmup // 2):
                e2e_ms.append(dt)
        e2e = {"value": statistics.mean(e2e_ms) / 1e3, "unit": "s",
               "h2d_bytes_per_step": esz * m * n_local + 16 * m, "d2h_bytes_per_step": 16 * n_local,
               "note": "wall clock around mnb_solve_randomized with host A (pinned) and host x"}
        if rank == 0:
            assert np.all(np.isfinite(rep_h.x))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # one complete CPU-port solve of the same instance (same bits as the device arm's A)
        if A_np is None:
            A_np = A.T.cpu().numpy().T
        threads = cpu_threads(cfg)
        dt, ref = cpu_solve(cfg, A_np, b, threads)
        cpu = cpu_record(dt, ref, threads, "1 solve")
        xg = rep_h.x if rep_h is not None else last.x.cpu().numpy()
        cpu["rel_x_gpu_vs_port"] = float(np.linalg.norm(xg - ref.x) / np.linalg.norm(ref.x))
        cpu["iterations_gpu_minus_port"] = last.lsq_iterations - ref.lsq_iterations
        one = recorded_single_thread(args.config)
        if one:
            cpu["single_thread"] = one

    # per-pass kernel time of the sketch and its algorithmic-bytes rate (fused pass when FA is 0)
    def gbs(bytes_per_elt, t_ms):
        return 2 * bytes_per_elt * m * n / (t_ms * 1e-3) / 1e9 if t_ms > 0 else None
    if sk[2] > 0:
        sketch_ms = {"hstage1": sk[0], "hstage2": sk[1], "fft_a": sk[2], "fft_b": sk[3]}
        sketch_gbs = {"hstage1": gbs(esz + 16, sk[0]), "hstage2": gbs(32, sk[1]), "fft_a": gbs(32, sk[2]),
                      "fft_b": gbs(16, sk[3])}
    else:
        sketch_ms = {"hstage1": sk[0], "hstage2+fft_a": sk[1], "fft_b": sk[3]}
        sketch_gbs = {"hstage1": gbs(esz + 16, sk[0]), "hstage2+fft_a": gbs(32, sk[1]), "fft_b": gbs(16, sk[3])}

    # The sketch against SURVEY 8(d)'s roofline: max(algorithmic bytes / HBM peak, FP64 flops / FP64
    # peak) over the measured device time of one sketch (CUDA events around each sketch in the solve).
    # Bytes: A once (16 or 8 B per entry) + the l x m output + ~88 B per index of parameters; flops:
    # m (5 n log2 n + 42 n) (the FFT of every row plus the two H chains, D and the diagonals).
    roofline_sketch = None
    sk_s = [t for t in last.extra["sketch_seconds"] if t > 0]
    if sk_s:
        l_ = 4 * m
        sk_bytes = esz * m * n + 16 * l_ * m + 88 * n
        sk_flops = m * (5.0 * n * math.log2(n) + 42.0 * n)
        fp64_peak, fp64_kind = fp64_peak_tfs()
        t_sk = statistics.mean(sk_s)
        t_hbm = sk_bytes / (hbm_peak * 1e9)
        t_fp = sk_flops / (fp64_peak * 1e12)
        fp_bound = t_fp >= t_hbm
        roofline_sketch = {
            "bound": "fp64" if fp_bound else "hbm",
            "achieved": (sk_flops / t_sk / 1e12) if fp_bound else (sk_bytes / t_sk / 1e9),
            "peak": fp64_peak if fp_bound else hbm_peak, "unit": "TFLOP/s" if fp_bound else "GB/s",
            "frac": max(t_hbm, t_fp) / t_sk, "ms_per_sketch": t_sk * 1e3,
            "floor_ms": {"hbm": t_hbm * 1e3, "fp64": t_fp * 1e3}, "peak_kind": {"hbm": peak_kind, "fp64": fp64_kind},
            "bytes_per_sketch": sk_bytes, "flops_per_sketch": sk_flops,
            "traffic": traffic_sketch if world == 1 else None,
            "note": "SURVEY 8(d): max(bytes/BW, flops/FP64) / measured sketch time (device events, in the solve); "
                    "traffic = ncu DRAM bytes of one sketch's kernels (P1, carries, fused P2 + pass A, pass B), "
                    "profiles/ncu_summary.json"}
        if sk[2] == 0 and sk[1] > 0:  # the fused H stage + FFT pass A alone, against the HBM peak
            per = 32 * m * n
            ach = 2 * per / (sk[1] * 1e-3) / 1e9
            roofline_sketch["p2fa_kernel"] = {"achieved": ach, "unit": "GB/s", "frac": ach / hbm_peak,
                                              "bytes_per_sketch": per, "ms_per_sketch": sk[1] / 2}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median": statistics.median(step_ms),
            "ms_per_step_all": step_ms, "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if cfg["real"] else "c128", "data": "synthetic (seeded, on device)",
            "config": config_json,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "kernel": "pcg_pass_kernel",
                         "peak_kind": peak_kind, "bytes_per_launch": pass_bytes, "ms_per_launch": pass_ms},
            **({"roofline_sketch": roofline_sketch} if roofline_sketch else {}),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            **({"classical": classical} if classical else {}),
            "solve": {"lsq_iterations": last.lsq_iterations, "lsq_converged": last.lsq_converged,
                      "residual_norm": last.residual_norm, "c_norm_ratio": last.c_norm_ratio,
                      "step_seconds": last.step_seconds, "param_seconds": last.extra["param_seconds"],
                      "total_seconds_host": last.extra.get("total_seconds"),
                      "sketch_seconds": last.extra["sketch_seconds"], "qr_seconds": last.extra["qr_seconds"],
                      "pcg_seconds": last.extra["pcg_seconds"],
                      "redistribute_seconds": last.extra["redistribute_seconds"],
                      "sketch_kernel_ms": sketch_ms, "sketch_hbm_gbs": sketch_gbs,
                      "note_sketch": "sketch_kernel_ms sums both sketches (S and E); GB/s = algorithmic bytes "
                                     "(read + write of one m x n pass) x 2 sketches / time; 'hstage2+fft_a' is "
                                     "the fused second H stage + FFT pass A (k_p2fa.cu: reads x1, writes pass A's "
                                     "output, 32 B per element)"},
        }
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
