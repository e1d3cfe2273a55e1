"""profiles/traffic_c2.json from an ncu raw CSV export (dram bytes per launch of the product kernels)."""
import csv
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
h = rows[0]
units = dict(zip(h, rows[1]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1, "us": 1e-3, "ns": 1e-6}
names = {"near_pair_kernel": "near_pairs", "t_pair_kernel": "lowrank_t", "rows_tma_kernel": "rows"}
out = {"source": "ncu --set full --clock-control none -k regex:'rows_tma|t_pair|near_pair' python bench.py --steps 2 "
                  "--warmup 1 (B200); dram__bytes_read.sum + dram__bytes_write.sum per launch",
       "config": {"n": 1048576, "d": 2, "c_leaf": 64, "k": 16, "mode": "stored", "near_sym": True}, "kernels": {}}
for r in rows[2:]:
    d = dict(zip(h, r))
    key = next((v for k, v in names.items() if k in d["Kernel Name"]), None)
    if not key or key in out["kernels"]:
        continue
    g = lambda m: float(d[m].replace(",", "")) * scale[units[m]]
    out["kernels"][key] = {"kernel": d["Kernel Name"].split("(")[0], "dram_read_bytes": g("dram__bytes_read.sum"),
                           "dram_write_bytes": g("dram__bytes_write.sum"),
                           "duration_ms": g("gpu__time_duration.sum")}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
