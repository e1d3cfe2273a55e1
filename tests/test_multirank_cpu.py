"""N > 1 host logic on CPU (gloo, world_size 2): every rank computes its row slice of the
product with the oracle's row-sampled evaluation (exactly the leaves the device rank
owns), the slices are all-gathered, and the result equals the single-process product
bitwise -- the property the row-cluster partition relies on."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_09707_b200.partition import row_slices, straddling_leaves


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, d, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bind import Oracle
    from paper_1708_09707_b200.inputs import symmetric, uniform_points
    O = Oracle()
    h = O.setup(uniform_points(n, d, 42), c_leaf=64, k=16)
    lo, hi = row_slices(n, world)[rank]
    x = symmetric(7, n)
    zm = h.mvp_rows(x, [(lo, hi)])
    from paper_1708_09707_b200.partition import allgather_rows
    full_m = allgather_rows(zm[lo:hi], n, world, rank)
    _, perm = h.points()
    z = np.empty(n)
    z[perm] = full_m
    if rank == 0:
        np.save(out_path, z)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,d", [(4096, 2), (3000, 3)])
def test_two_rank_product_equals_single(tmp_path, oracle, n, d):
    from paper_1708_09707_b200.inputs import symmetric, uniform_points
    out = str(tmp_path / "z.npy")
    mp.spawn(_worker, args=(2, _free_port(), n, d, out), nprocs=2, join=True)
    z2 = np.load(out)
    z1 = oracle.setup(uniform_points(n, d, 42), c_leaf=64, k=16).mvp(symmetric(7, n))
    assert np.array_equal(z2.view(np.uint64), z1.view(np.uint64))


@pytest.mark.parametrize("n,d,world", [(1 << 14, 2, 8), (1 << 14, 3, 8), (1 << 13, 2, 4), (5000, 2, 2)])
def test_no_leaf_straddles_the_partition(oracle, n, d, world):
    from paper_1708_09707_b200.inputs import uniform_points
    h = oracle.setup(uniform_points(n, d, 42), c_leaf=64, k=16)
    for which in (0, 1):
        assert straddling_leaves(h.leaves(which, boxes=False).rows, n, world) == []


def test_row_slices_tile_the_rows():
    for n in (1000, 4096, 12345):
        for world in (1, 2, 4, 8):
            sl = row_slices(n, world)
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        row_slices(100, 3)
