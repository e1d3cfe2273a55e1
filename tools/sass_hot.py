"""Aggregate an ncu --page source --print-source sass CSV: executed instructions and
stall samples per opcode, and the hottest instruction ranges.
usage: python tools/sass_hot.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
ops = defaultdict(lambda: [0, 0])
tot_inst = tot_samp = 0
for r in data:
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ie = int(r[ix["Instructions Executed"]] or 0)
    sm = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ops[op][0] += ie
    ops[op][1] += sm
    tot_inst += ie
    tot_samp += sm
print(f"total warp-instructions {tot_inst:.4g}, samples {tot_samp}")
for op, (ie, sm) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:28]:
    print(f"  {op:10s} inst {ie / tot_inst * 100:5.1f}%   samples {sm / max(tot_samp, 1) * 100:5.1f}%")
# hottest windows of 32 consecutive instructions by samples
top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
win = 48
sc = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
best = sorted(((sum(sc[i:i + win]), i) for i in range(0, len(sc), win)), reverse=True)[:top]
for s, i in best:
    ie = sum(int(r[ix["Instructions Executed"]] or 0) for r in data[i:i + win])
    print(f"--- window @{i} samples {s / max(tot_samp, 1) * 100:.1f}% inst {ie / tot_inst * 100:.1f}%")
    for r in data[i:i + win]:
        if int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) * 400 > tot_samp or int(r[ix["Instructions Executed"]] or 0) * 300 > tot_inst:
            print(f"   {r[ix['Source']].strip()[:70]:72s} inst {int(r[ix['Instructions Executed']] or 0):>11d} samp {r[ix['Warp Stall Sampling (All Samples)']]}")
# top single instructions with their dominant stall reasons
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("--- top instructions")
order = sorted(range(len(data)), key=lambda i: -sc[i])[:top * 3]
for i in order:
    r = data[i]
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"   @{i:5d} {r[ix['Source']].strip()[:60]:62s} samp {sc[i] / max(tot_samp, 1) * 100:4.1f}%  " +
          " ".join(f"{n}:{v}" for v, n in st if v))
