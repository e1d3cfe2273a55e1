# Build-phase trace at a bench configuration (HM_TRACE=1 prints device phase times).
import os, sys, time
sys.path.insert(0, '.')
os.environ.setdefault("HM_TRACE", "1")
import paper_1708_09707_b200 as hm
from paper_1708_09707_b200.inputs import uniform_points
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
d = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kern = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
P = uniform_points(n, d, 42)
for rep in range(2):
    t = time.perf_counter()
    h = hm.setup(P, hm.KernelFunction(kern), hm.HmatrixConfig(c_leaf=64, k=16, precompute_aca=True, near_stored=True))
    print("setup", time.perf_counter() - t, h.timings(), flush=True)
    del h
