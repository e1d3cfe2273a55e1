# one recompute product at N=2^18 d=4 (for ncu captures of the ACA kernels in the clean regime)
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_09707_b200 as hm
from paper_1708_09707_b200.inputs import symmetric, uniform_points
n = 1 << 18
h = hm.setup(uniform_points(n, 4, 42), hm.KernelFunction(), hm.HmatrixConfig(c_leaf=64, k=16))
h.mvp(symmetric(43, n))
