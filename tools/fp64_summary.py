"""Turns the ncu CSV of tools/c_eval.py (+ tools/fp64_peak output) into
profiles/fp64_peaks.json: c_eval per kernel/dimension (FP64 thread-instructions per
entry) and the measured FP64 instruction throughput (the FP64 roofline denominator).

  python tools/fp64_summary.py <ncu_c_eval.csv> <fp64_peak.json> > profiles/fp64_peaks.json
"""
import csv
import json
import sys

N = 1 << 22
ORDER = [("gaussian", 2), ("gaussian", 3), ("gaussian", 4), ("matern", 2), ("matern", 3), ("matern", 4)]


def main():
    rows = []
    with open(sys.argv[1]) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per = {}
    for r in rows:
        per.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ids = sorted(per)
    assert len(ids) == len(ORDER), (len(ids), ids)
    c_eval, detail = {}, {}
    for (kern, d), i in zip(ORDER, ids):
        m = per[i]
        dfma = m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
        dadd = m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
        dmul = m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
        fp64 = m.get("smsp__sass_thread_inst_executed_op_fp64_pred_on.sum", dfma + dadd + dmul)
        key = f"{kern}_d{d}"
        c_eval[key] = fp64 / N
        detail[key] = {"dfma": dfma / N, "dadd": dadd / N, "dmul": dmul / N, "fp64_all": fp64 / N,
                       "flop": (2 * dfma + dadd + dmul) / N}
    with open(sys.argv[2]) as f:
        peak = json.loads([ln for ln in f if ln.startswith("{")][-1])
    out = {"what": "FP64 roofline constants measured on the B200 box: c_eval = FP64-pipe thread-instructions "
                   "per kernel entry (ncu smsp__sass_thread_inst_executed_op_fp64_pred_on over 2^22 random "
                   "pairs in [0,1]^d, tools/c_eval.py); fp64_inst_per_s = DFMA thread-instruction throughput "
                   "(tools/fp64_peak.cu, all SMs, 8 independent chains per thread)",
           "c_eval": c_eval, "c_eval_detail": detail, "fp64_inst_per_s": peak["dfma_inst_per_s"],
           "peak_detail": peak}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
