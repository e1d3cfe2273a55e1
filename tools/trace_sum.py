"""Per-class ACA device time summed over a HM_TRACE log (stderr of bench.py / one_product.py).
usage: python tools/trace_sum.py log [log ...]"""
import collections
import re
import sys

for f in sys.argv[1:]:
    T = collections.defaultdict(float)
    for ln in open(f):
        m = re.match(r"\[hm_trace\] (.+?)\s{2,}([\d.]+) ms", ln)
        if m and not ln.startswith("[hm_trace] plan"):
            T[m.group(1).strip()] += float(m.group(2))
    tot = sum(T.values())
    print(f, f"total {tot:.0f} ms")
    for k, v in T.items():
        print(f"  {k:28s} {v:9.1f} ms  {100 * v / tot:5.1f}%")
