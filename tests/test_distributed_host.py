"""CPU tests of the slab decomposition's host logic:
partition, owned/halo selection against a brute-force neighbour check, and
the rank-ordered collectives over a world-size-2 gloo group."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_01754_b200.distributed import TorchComm, leaf_x, select_local, slab_partition, wrap


@pytest.mark.parametrize("depth,world", [(3, 1), (3, 2), (4, 4), (4, 8), (5, 8), (1, 2)])
def test_slab_partition_covers_grid(depth, world):
    lg, ranges = slab_partition(depth, world)
    assert 2 ** lg == world
    n = 2 ** depth
    covered = np.concatenate([np.arange(a, b) for a, b in ranges])
    assert np.array_equal(covered, np.arange(n))
    assert len({b - a for a, b in ranges}) == 1


def test_slab_partition_rejects_bad_worlds():
    with pytest.raises(ValueError):
        slab_partition(3, 3)
    with pytest.raises(ValueError):
        slab_partition(2, 8)


@pytest.mark.parametrize("depth,world", [(3, 2), (3, 4), (4, 8), (2, 4)])
def test_owned_plus_halo_hold_every_p2p_source(depth, world):
    rng = np.random.default_rng(depth * 10 + world)
    box = 3.0
    pos = wrap(rng.uniform(-1, 4, size=(4000, 3)), box)
    lx = leaf_x(pos, box, depth)
    n = 2 ** depth
    _, ranges = slab_partition(depth, world)
    seen = np.zeros(len(pos), int)
    for x0, x1 in ranges:
        own, halo = select_local(lx, x0, x1, depth)
        seen[own] += 1
        assert not np.intersect1d(own, halo).size
        # every neighbour leaf plane of an owned leaf (periodic) is present
        have = np.zeros(n, bool)
        have[np.unique(lx[np.concatenate([own, halo])])] = True
        for x in range(x0, x1):
            for dx in (-1, 0, 1):
                xs = (x + dx) % n
                if np.any(lx == xs):
                    assert have[xs]
    assert np.all(seen == 1)


def test_leaf_x_matches_octree_assignment():
    from oracle import lfmm_oracle as orc

    rng = np.random.default_rng(3)
    box = 2.5
    pos = wrap(rng.uniform(0, box, size=(500, 3)), box)
    tree = orc.build_tree(pos, box, 3)
    leaf = tree["leaf_of_particle"][tree["inv_perm"]]
    assert np.array_equal(leaf_x(pos, box, 3), leaf // 64)


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        # in-place all-gather of rank-owned chunks
        buf = torch.zeros(world * 3, dtype=torch.float64)
        buf[rank * 3:(rank + 1) * 3] = torch.tensor([rank + 1.0, rank + 2.0, rank + 3.0])
        comm.allgather_(buf, 3)
        # rank-ordered sum: the same bits on every rank
        t = torch.tensor([0.1 * (rank + 1), 1e16, -1e16 + rank], dtype=torch.float64)
        s = comm.sum_ordered(t)
        out_q.put((rank, buf.numpy().copy(), s.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_torch_comm_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (b, s)) for r, b, s in [q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    expect = np.array([1, 2, 3, 2, 3, 4], float)
    for r in range(2):
        assert np.array_equal(res[r][0], expect)
    assert res[0][1].tobytes() == res[1][1].tobytes()
    ref = np.array([0.1, 1e16, -1e16]) + np.array([0.2, 1e16, -1e16 + 1])
    assert np.allclose(res[0][1], ref)
