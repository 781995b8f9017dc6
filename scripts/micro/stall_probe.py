"""Where do multi-ms host stalls come from on the GPU box?  (1) a CPU spin loop
records gaps > 1 ms between clock reads (vCPU preemption / steal); (2) tiny
kernel + synchronize round trips record driver-side latency outliers."""
import time, threading, sys
import torch

def spin(sec, out):
    gaps = []
    t_end = time.perf_counter() + sec
    prev = time.perf_counter()
    while prev < t_end:
        now = time.perf_counter()
        if now - prev > 1e-3:
            gaps.append(round((now - prev) * 1e3, 2))
        prev = now
    out.append(gaps)

for label, nthreads in (("1 spinner", 1), ("8 spinners", 8)):
    outs = []
    ths = [threading.Thread(target=spin, args=(5.0, outs)) for _ in range(nthreads)]
    [t.start() for t in ths]; [t.join() for t in ths]
    allg = sorted(g for o in outs for g in o)
    print(label, "gaps>1ms:", len(allg), "max", allg[-5:] if allg else [], flush=True)

x = torch.zeros(16, device="cuda")
torch.cuda.synchronize()
lat = []
t_end = time.perf_counter() + 10
while time.perf_counter() < t_end:
    t = time.perf_counter(); x.add_(1); torch.cuda.synchronize(); lat.append((time.perf_counter() - t) * 1e3)
lat.sort()
print("launch+sync round trips:", len(lat), "median %.3f ms p99 %.3f max %s" % (lat[len(lat)//2], lat[int(len(lat)*0.99)], [round(v, 1) for v in lat[-8:]]), flush=True)
# same while the spinner runs in another thread (GIL contention aside)
big = torch.empty(1 << 28, device="cuda")
lat = []
t_end = time.perf_counter() + 10
while time.perf_counter() < t_end:
    t = time.perf_counter(); big.mul_(1.0); torch.cuda.synchronize(); lat.append((time.perf_counter() - t) * 1e3)
lat.sort()
print("1 GiB elementwise round trips:", len(lat), "median %.3f ms p99 %.3f max %s" % (lat[len(lat)//2], lat[int(len(lat)*0.99)], [round(v, 1) for v in lat[-8:]]), flush=True)
