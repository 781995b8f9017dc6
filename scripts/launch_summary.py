"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel count / total / share, keeping only the solve steps after warm-up
(launches after the last 'mark' kernel when given).  usage:
python scripts/launch_summary.py launches.csv [--last-fraction F]"""
import csv, io, sys, re
from collections import OrderedDict

path = sys.argv[1]
txt = open(path).read()
i = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[i:])))
agg = OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"(?:mnb::)?(?:<unnamed>::|unnamed>::)?([A-Za-z0-9_]+)(?:<[^(]*>)?\(", name)
    key = m.group(1) if m else name[:60]
    if "mnb" not in name and "unnamed" not in name:
        key = "lib:" + key
    ns = float(r["Metric Value"].replace(",", ""))
    c, t = agg.get(key, (0, 0.0))
    agg[key] = (c + 1, t + ns)
tot = sum(t for c, t in agg.values())
print(f"{'kernel':40s} {'launches':>9s} {'total ms':>10s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:40]:40s} {c:9d} {t / 1e6:10.3f} {t / tot * 100:6.1f}%")
print(f"{'TOTAL':40s} {sum(c for c, t in agg.values()):9d} {tot / 1e6:10.3f}")
