"""Summarise an ncu report: key throughput metrics, stall reasons, opcode mix.
usage: python scripts/ncu_summary.py report.ncu-rep [kernel-substring]"""
import csv, io, re, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = [r'gpu__time_duration.sum$', r'dram__bytes_read.sum$', r'dram__bytes_write.sum$',
        r'dram__throughput.avg.pct_of_peak_sustained_elapsed$', r'smsp__inst_executed.sum$',
        r'sm__issue_active.avg.pct_of_peak_sustained_elapsed$', r'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active$',
        r'launch__registers_per_thread$', r'launch__grid_size$', r'launch__block_size$',
        r'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$', r'lts__t_sector_hit_rate.pct$',
        r'smsp__pcsamp_warps_issue_stalled_(?!.*not_issued)']
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("kernel:", d.get("Kernel Name", "")[:120])
    for k, v in d.items():
        if any(re.search(p, k) for p in keys) and v not in ("0", "0.000000", ""):
            print(f"  {k} = {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
try:
    i0 = next(i for i, r in enumerate(srows) if r and r[0] == "Address")
    h = srows[i0]
    ie = h.index("Instructions Executed")
    tot = 0; c = Counter()
    for r in srows[i0 + 1:]:
        if len(r) > ie and r[ie].isdigit():
            n = int(r[ie]); tot += n
            t = r[1].strip().split()
            if not t: continue
            op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
            c[op.split(".")[0]] += n
    print("  opcode mix (% of executed warp instructions):",
          ", ".join(f"{o} {n / tot * 100:.1f}" for o, n in c.most_common(14)))
except StopIteration:
    pass
