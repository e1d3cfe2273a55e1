"""Summarise ncu CSV exports: key metrics per kernel + SASS opcode mix / top stalls."""
import csv
import sys
from collections import Counter, defaultdict

KEYS = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput",
        "Memory Throughput", "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction", "Block Limit Registers",
        "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]


def details(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    out = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = (d.get("ID"), d["Kernel Name"][:90])
        out[k][d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    for k, m in out.items():
        print("==", k[1])
        for key in KEYS:
            if key in m:
                print(f"   {key:40s} {m[key][0]} {m[key][1]}")


def sass(path, top=20):
    rows = list(csv.reader(open(path)))
    # possibly several kernels: split on "Kernel Name" header lines
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["h"] = r
        elif cur is not None and "h" in cur and len(r) >= len(cur["h"]):
            cur["rows"].append(r)
    for b in blocks:
        h = b["h"]
        iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        data = []
        for r in b["rows"]:
            try:
                data.append((r[iS].strip(), int(r[iW]), int(r[iE])))
            except ValueError:
                pass
        te = sum(d[2] for d in data) or 1
        ts = sum(d[1] for d in data) or 1
        c, cs = Counter(), Counter()
        for s, w, e in data:
            tok = s.split()
            op = tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "?")
            op = op.split(".")[0]
            c[op] += e
            cs[op] += w
        print("==", b["name"][:100], "executed", te)
        print("   " + "  ".join(f"{op}:{v / te * 100:.1f}%/{cs[op] / ts * 100:.1f}%" for op, v in c.most_common(top)))
        for s, w, e in sorted(data, key=lambda x: -x[1])[:top]:
            print(f"   stall {w / ts * 100:5.2f}%  exec {e:>12d}  {s[:90]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        (sass if p.endswith("_sass.csv") else details)(p)
