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


def allgather_rows(mine, n: int, world: int, rank: int, group=None):
    """Host-transport allgather of the y row slices (the gloo / CPU path of the NCCL
    y-allgather in hm_api.cu, allgather_y): every rank contributes its Morton rows
    [lo, hi) of row_slices(n, world) and receives the full Morton-ordered vector.
    Slices may differ by one row (ceil splits): they are padded to the widest."""
    import numpy as np
    import torch
    import torch.distributed as dist
    bounds = row_slices(n, world)
    lo, hi = bounds[rank]
    mine = np.asarray(mine, dtype=np.float64)
    if mine.shape != (hi - lo,):
        raise ValueError("allgather_rows: slice length does not match the rank's rows")
    width = max(b - a for a, b in bounds)
    padded = torch.zeros(width, dtype=torch.float64)
    padded[: hi - lo] = torch.from_numpy(mine)
    gathered = [torch.empty(width, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, padded, group=group)
    return np.concatenate([gathered[r][: b - a].numpy() for r, (a, b) in enumerate(bounds)])
