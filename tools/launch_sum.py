"""Sum an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name.
usage: python tools/launch_sum.py launches.csv [top]"""
import csv
import sys
from collections import defaultdict

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
tot = defaultdict(lambda: [0.0, 0])
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    unit = r.get("Metric Unit", "ns")
    v = float(r["Metric Value"].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6,
                                                     "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    tot[name][0] += v
    tot[name][1] += 1
all_ms = sum(v[0] for v in tot.values())
print(f"total {all_ms:.1f} ms over {sum(v[1] for v in tot.values())} launches")
for name, (ms, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"  {ms:10.2f} ms  {ms / all_ms * 100:5.1f}%  x{c:<5d} {name[:90]}")
