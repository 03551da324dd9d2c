"""World-size-2 gloo run of the bench's multi-rank plumbing (replica seeding,
barrier, max-over-ranks timing) on CPU."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    r, w, l = bench.dist_env()
    assert (r, w, l) == (rank, world, rank)
    # each rank times a different amount of work; the reported time is the max
    t = torch.tensor([10.0 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out[rank] = float(t.item())
    # replicas use seed + rank
    class A:
        atoms, sites, seed = 600, 2, 7
    sysA, _ = bench.load_system(A, rank)
    h = torch.tensor([float(sysA.positions.sum())], dtype=torch.float64)
    hs = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(hs, h)
    out[10 + rank] = float(hs[0].item() != hs[1].item())
    dist.destroy_process_group()


def test_two_rank_gloo_max_and_replicas():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == out[1] == 20.0
    assert out[10] == 1.0 and out[11] == 1.0
