"""CPU tests of the slab decomposition's host logic:
partition, owned/halo selection against a brute-force neighbour check, and
the rank-ordered collectives over a world-size-2 gloo group."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_01754_b200.distributed import (TorchComm, _halo_ops, halo_planes, leaf_x, select_local,
                                               slab_partition, wrap)


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


@pytest.mark.parametrize("depth,world,level", [(4, 2, 4), (4, 4, 3), (4, 8, 4), (5, 8, 5), (6, 4, 6)])
def test_halo_ops_deliver_every_m2l_source_plane(depth, world, level):
    """The planes each rank receives are exactly the M2L source planes of its
    owned targets outside its slab (children of the parents' neighbours:
    x in [2(px-1), 2(px+1)+1], octree.py:96-111), and every receive is
    matched by the owning neighbour's send, in order, per peer."""
    lg, ranges = slab_partition(depth, world)
    n = 1 << level
    sh = depth - level
    sends, recvs = {}, {}
    for r, (a, b) in enumerate(ranges):
        x0, x1 = a >> sh, b >> sh
        need = set()
        for x in range(x0, x1):
            px = x // 2
            need |= {(2 * (px + dp) + c) % n for dp in (-1, 0, 1) for c in (0, 1)}
        need -= set(range(x0, x1))
        assert set(halo_planes(x0, x1, n)) == need
        for kind, peer, first in _halo_ops(r, world, x0, x1, n):
            if kind == "send":
                sends.setdefault((r, peer), []).append(first)
            else:
                pa, pb = ranges[peer]
                assert pa >> sh <= first and first + 2 <= pb >> sh, "received planes are owned by the peer"
                recvs.setdefault((peer, r), []).append(first)
    assert sends == recvs


def _halo_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        n, plane = 16, 5
        w = n // world
        x0, x1 = rank * w, (rank + 1) * w
        buf = torch.full((n * plane,), -1.0, dtype=torch.float64)
        for x in range(x0, x1):
            buf[x * plane:(x + 1) * plane] = 100.0 * x + torch.arange(plane, dtype=torch.float64)
        comm.halo_(buf, plane, x0, x1, n)
        m = torch.tensor([rank, 10 - rank, 7], dtype=torch.int32)
        comm.max_(m)
        out_q.put((rank, buf.numpy().copy(), m.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_torch_comm_halo_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + world + (os.getpid() % 1000)
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (b, m)) for r, b, m in [q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    n, plane = 16, 5
    w = n // world
    for r in range(world):
        x0, x1 = r * w, (r + 1) * w
        filled = set(range(x0, x1)) | set(halo_planes(x0, x1, n))
        buf = res[r][0].reshape(n, plane)
        for x in range(n):
            if x in filled:
                assert np.array_equal(buf[x], 100.0 * x + np.arange(plane))
            else:
                assert np.all(buf[x] == -1.0)
        assert list(res[r][1]) == [world - 1, 10, 7]


def _particle_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_01754_b200.distributed import DistributedSolver
        from paper_2410_01754_b200.fmm.solver import SolverConfig

        depth, box = 3, 3.0
        rng = np.random.default_rng(0)
        pos = rng.uniform(-1, 4, size=(3000, 3))
        moved = pos + rng.uniform(-0.3, 0.3, size=pos.shape)
        solver = DistributedSolver(box, SolverConfig(p=4, depth=depth), comm=TorchComm())
        lx = leaf_x(wrap(pos, box), box, depth)
        own = np.flatnonzero((lx >= solver.x0) & (lx < solver.x1))
        p_l, q_l, g_l, n_own = solver._exchange_particles(torch.from_numpy(moved[own]),
                                                          torch.from_numpy(own * 0.5),
                                                          torch.from_numpy(own.astype(np.int64)))
        out_q.put((rank, p_l.numpy(), q_l.numpy(), g_l.numpy(), n_own, moved))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_particle_halo_exchange_gloo(world):
    """After the exchange each rank holds exactly the atoms select_local
    picks from the global moved positions: owned = its slab, halo = the
    leaf planes either side, with their positions, charges and ids."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + world + (os.getpid() % 1000)
    procs = [ctx.Process(target=_particle_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: rest for r, *rest in [q.get(timeout=120) for _ in procs]}
    for p in procs:
        p.join(timeout=60)
    depth, box = 3, 3.0
    _, ranges = slab_partition(depth, world)
    for r, (x0, x1) in enumerate(ranges):
        p_l, q_l, g_l, n_own, moved = res[r]
        lx = leaf_x(wrap(moved, box), box, depth)
        own, halo = select_local(lx, x0, x1, depth)
        assert sorted(g_l[:n_own]) == sorted(own)
        assert sorted(g_l[n_own:]) == sorted(halo)
        assert np.array_equal(p_l, moved[g_l])
        assert np.array_equal(q_l, g_l * 0.5)


def test_single_plane_slabs_reject_migrants():
    """with one leaf plane per rank (depth 2, world 4) a migrant
    into plane x1 is also rank r+2's halo, which the one-hop exchange never
    reaches; step_owned must refuse instead of dropping P2P pairs."""
    import torch

    from paper_2410_01754_b200.distributed import DistributedSolver, LocalComm
    from paper_2410_01754_b200.fmm.solver import SolverConfig

    box, depth, world = 4.0, 2, 4
    solver = DistributedSolver(box, SolverConfig(p=4, depth=depth), comm=LocalComm(world).for_rank(1))
    assert (solver.x0, solver.x1) == (1, 2)
    pos = torch.tensor([[1.5, 0.3, 0.3], [1.2, 2.0, 1.0], [0.5, 1.0, 1.0]], dtype=torch.float64)  # last: plane 0
    q = torch.zeros(3, dtype=torch.float64)
    gid = torch.arange(3)
    with pytest.raises(ValueError, match="single leaf plane"):
        solver._exchange_particles(pos, q, gid)


def test_sites_without_lambdas_rejected():
    """sites given without lambdas would run the HI kernel on
    never-uploaded lambdas; the step refuses before any device work."""
    import torch

    from paper_2410_01754_b200.distributed import DistributedSolver, LocalComm
    from paper_2410_01754_b200.fmm.solver import SolverConfig

    solver = DistributedSolver(4.0, SolverConfig(p=4, depth=2), comm=LocalComm(1).for_rank(0))
    pos = torch.rand(8, 3, dtype=torch.float64) * 4.0
    tables = (np.array([0, 2]), np.array([0, 1]), np.array([2], np.int32), np.array([0, 4]), np.zeros(4))
    with pytest.raises(ValueError, match="lambdas"):
        solver._step(pos, torch.zeros(8, dtype=torch.float64), torch.arange(8), None, None, tables, 8, 0)
