"""The whole slab-decomposed step (DistributedSolver.step) over a real
torch.distributed group: two processes, gloo backend (collectives staged
through host memory), both on cuda:0 of the one-GPU test box.  Energy, every
owned force row and every site's lambda forces must reproduce the single-GPU
lfmm_step; the NCCL backend runs the same TorchComm code on
device tensors."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, precision, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2410_01754_b200.distributed import DistributedSolver, TorchComm
        from paper_2410_01754_b200.fmm.solver import SolverConfig
        from paper_2410_01754_b200.system import lambda_table, site_tables
        from paper_2410_01754_b200.waterbox import generate_water_box

        system, lam, _ = generate_water_box(40_000, 24, seed=11)
        cfg = SolverConfig(p=10, depth=4, precision=precision)
        dev = torch.device("cuda", 0)
        lt, nl = lambda_table(system, lam.values)
        solver = DistributedSolver(system.box_length, cfg, comm=TorchComm())
        out = solver.step(torch.from_numpy(system.positions).to(dev), torch.from_numpy(system.charges).to(dev),
                          torch.from_numpy(lt).to(dev), torch.from_numpy(nl).to(dev), sites=site_tables(system))
        torch.cuda.synchronize()
        out_q.put((rank, out["energy"], out["owned"].cpu().numpy(), out["forces"].cpu().numpy(),
                   out["lambda_forces"].cpu().numpy()))
    except Exception as e:  # surfaced by the parent
        out_q.put((rank, repr(e), None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["double", "single"])
def test_distributed_step_over_gloo_matches_single_gpu(precision):
    import multiprocessing as mp

    from paper_2410_01754_b200 import _native
    from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig
    from paper_2410_01754_b200.system import lambda_table, site_tables
    from paper_2410_01754_b200.waterbox import generate_water_box

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 32500 + (os.getpid() % 1000) + (7 if precision == "single" else 0)
    procs = [ctx.Process(target=_worker, args=(r, world, port, precision, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: rest for r, *rest in [q.get(timeout=600) for _ in procs]}
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert res[r][1] is not None, res[r][0]

    system, lam, _ = generate_water_box(40_000, 24, seed=11)
    cfg = SolverConfig(p=10, depth=4, precision=precision)
    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    plan = solver.plan
    plan.set_sites(*site_tables(system))
    lt, nl = lambda_table(system, lam.values)
    e = np.empty(1)
    f = np.empty((system.num_particles, 3))
    lf = np.empty((len(system.sites), 4))
    plan.step(system.positions, system.charges, lt, nl, mode=_native.MODE_HI, energy=e, forces=f, lambda_forces=lf)
    tol = 1e-10 if precision == "double" else 1e-6
    forces = np.full_like(f, np.nan)
    for r in range(world):
        energy, owned, fr, lfr = res[r]
        assert abs(energy - e[0]) <= tol * abs(e[0])
        forces[owned] = fr
        assert np.max(np.abs(lfr - lf)) <= tol * np.max(np.abs(lf))
    assert not np.isnan(forces).any(), "every atom is owned by one rank"
    assert np.max(np.abs(forces - f)) <= tol * np.max(np.abs(f))
