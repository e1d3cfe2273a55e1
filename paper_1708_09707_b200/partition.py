"""Row-cluster ownership across ranks, host-side mirror.

Rank g of G = 2^q ranks owns the Morton rows of the depth-q cluster g of the implicit
cardinality-split cluster tree (first child gets ceil(size/2), proj/src/tree.cpp:120-123).
Every block-tree leaf lies at depth >= q for the benchmark configurations,
so each leaf -- hence each row's whole accumulation -- belongs to exactly one rank and
the row slices concatenate to the single-GPU product bitwise.  The C++ engine computes
the same bounds on the device (setup.cu, build_hmatrix)."""
from __future__ import annotations


def cluster_range(n: int, depth: int, idx: int):
    lo, hi = 0, n
    for b in range(depth - 1, -1, -1):
        mid = lo + (hi - lo + 1) // 2
        if (idx >> b) & 1:
            lo = mid
        else:
            hi = mid
    return lo, hi


def row_slices(n: int, world: int):
    q = world.bit_length() - 1
    if world < 1 or (1 << q) != world:
        raise ValueError("world size must be a power of two")
    return [cluster_range(n, q, g) for g in range(world)]


def straddling_leaves(rows4, n: int, world: int):
    """Leaves whose row cluster crosses a rank boundary (must be empty)."""
    bounds = row_slices(n, world)
    bad = []
    for (rl, ru, cl, cu) in rows4:
        for lo, hi in bounds:
            if rl < hi and lo < ru and (rl < lo or ru > hi):
                bad.append((rl, ru, cl, cu))
                break
    return bad
