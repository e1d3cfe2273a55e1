"""Summarise an ncu --page raw CSV: per kernel duration, FP64 pipe %, issue %, warps, and
the top warp-stall reasons (pc sampling).  usage: python tools/ncu_stalls.py raw.csv"""
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rd = list(csv.reader(lines))
hdr, data = rd[0], rd[2:]
ix = {h: i for i, h in enumerate(hdr)}


def g(row, name):
    try:
        return float(row[ix[name]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
for row in data:
    name = row[ix["Kernel Name"]][:70]
    print(f"{name}\n  dur {g(row, 'gpu__time_duration.sum') / 1e6:.2f} ms  fp64pipe "
          f"{g(row, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%  fp64inst "
          f"{g(row, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f}%  issue "
          f"{g(row, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}%  warps "
          f"{g(row, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%  regs {g(row, 'launch__registers_per_thread'):.0f}"
          f"  inst {g(row, 'smsp__inst_executed.sum'):.3g}")
    tot = sum(g(row, h) for h in stall if g(row, h) == g(row, h))
    top = sorted(((g(row, h), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stall
                  if g(row, h) == g(row, h)), reverse=True)[:7]
    print("  stalls: " + ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in top if tot))
