"""Slab-decomposed step on one GPU: G ranks simulated as
threads (LocalComm) must reproduce the single-GPU step — energy, every
atom's force, every site's lambda forces — since each box's multipoles, M2L
and P2P are computed as on one GPU and every reduction adds rank partials in
rank order."""

import threading

import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu

from paper_2410_01754_b200 import _native  # noqa: E402
from paper_2410_01754_b200.distributed import DistributedSolver, LocalComm  # noqa: E402
from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig  # noqa: E402
from paper_2410_01754_b200.system import lambda_table, site_tables  # noqa: E402
from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402


@pytest.fixture(scope="module")
def wb():
    system, lam, _ = generate_water_box(40_000, 24, seed=11)
    return system, lam


def _single(system, lam_values, cfg):
    s = PeriodicSolver(system.positions, system.box_length, cfg)
    plan = s.plan
    plan.set_sites(*site_tables(system))
    lam, nl = lambda_table(system, lam_values)
    n = system.num_particles
    e = np.empty(1)
    f = np.empty((n, 3))
    lf = np.empty((len(system.sites), 4))
    plan.step(system.positions, system.charges, lam, nl, mode=_native.MODE_HI, energy=e, forces=f,
              lambda_forces=lf)
    return float(e[0]), f, lf


def _distributed(system, lam_values, cfg, world):
    import torch

    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(np.ascontiguousarray(system.positions)).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(system.charges)).to(dev)
    lam, nl = lambda_table(system, lam_values)
    d_lam = torch.from_numpy(lam).to(dev)
    d_nl = torch.from_numpy(nl).to(dev)
    tables = site_tables(system)
    site_pos = pos[torch.from_numpy(tables[1]).to(dev)].contiguous()
    shared = LocalComm(world)
    outs = [None] * world
    errs = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            solver = DistributedSolver(system.box_length, cfg, comm=shared.for_rank(rank))
            outs[rank] = solver.step(pos, q, d_lam, d_nl, sites=tables, site_positions=site_pos)
            torch.cuda.synchronize()
        except Exception as e:  # surfaced below
            errs.append(e)
            shared.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    n = system.num_particles
    forces = np.zeros((n, 3))
    count = np.zeros(n, int)
    for o in outs:
        idx = o["owned"].cpu().numpy()
        forces[idx] = o["forces"].cpu().numpy()
        count[idx] += 1
    assert np.all(count == 1), "every atom is owned by exactly one rank"
    return outs, forces


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_slab_decomposition_matches_single_gpu(wb, precision, world):
    system, lam = wb
    cfg = SolverConfig(p=10, depth=4, precision=precision)
    e1, f1, lf1 = _single(system, lam.values, cfg)
    outs, fd = _distributed(system, lam.values, cfg, world)
    tol = 1e-10 if precision == "double" else 1e-6
    energies = [o["energy"] for o in outs]
    assert len(set(energies)) == 1, "every rank reports the same energy"
    assert abs(energies[0] - e1) <= tol * abs(e1)
    assert relerr(fd, f1) <= tol
    for o in outs:
        assert relerr(o["lambda_forces"].cpu().numpy(), lf1) <= tol


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_multipole_halo_exchange_reads_only_the_halo(wb, precision, world, monkeypatch):
    """Levels above lg exchange only the 2-plane multipole halo: every plane
    the exchange did not fill is set to NaN before phase 2, and the step
    still reproduces the single-GPU forces and lambda forces."""
    from paper_2410_01754_b200 import distributed

    monkeypatch.setattr(distributed, "_POISON", True)
    system, lam = wb
    cfg = SolverConfig(p=10, depth=4, precision=precision)
    e1, f1, lf1 = _single(system, lam.values, cfg)
    outs, fd = _distributed(system, lam.values, cfg, world)
    tol = 1e-10 if precision == "double" else 1e-6
    assert np.all(np.isfinite(fd))
    assert abs(outs[0]["energy"] - e1) <= tol * abs(e1)
    assert relerr(fd, f1) <= tol
    for o in outs:
        assert relerr(o["lambda_forces"].cpu().numpy(), lf1) <= tol


@pytest.mark.parametrize("world", [2, 4])
def test_step_owned_hands_over_migrated_atoms(wb, world):
    """Each rank starts from the atoms it owned before the atoms moved (up to
    0.2 nm, less than a leaf edge); atoms that crossed into a neighbour's
    slab are handed over in the halo exchange and the step equals the
    single-GPU step on the moved positions."""
    import torch

    from paper_2410_01754_b200.distributed import leaf_x, slab_partition, wrap

    system, lam = wb
    cfg = SolverConfig(p=10, depth=4, precision="double")
    rng = np.random.default_rng(5)
    moved = system.positions + rng.uniform(-0.2, 0.2, size=system.positions.shape)
    lx_old = leaf_x(wrap(system.positions, system.box_length), system.box_length, 4)
    lx_new = leaf_x(wrap(moved, system.box_length), system.box_length, 4)
    _, ranges = slab_partition(4, world)
    assert any(((lx_old >= a) & (lx_old < b)).sum() != ((lx_new >= a) & (lx_new < b)).sum() for a, b in ranges)
    import copy

    msys = copy.copy(system)
    msys.positions = moved
    e1, f1, lf1 = _single(msys, lam.values, cfg)

    dev = torch.device("cuda", 0)
    lam_t, nl = lambda_table(system, lam.values)
    d_lam = torch.from_numpy(lam_t).to(dev)
    d_nl = torch.from_numpy(nl).to(dev)
    tables = site_tables(system)
    shared = LocalComm(world)
    outs = [None] * world
    errs = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            a, b = ranges[rank]
            own = np.flatnonzero((lx_old >= a) & (lx_old < b))
            solver = DistributedSolver(system.box_length, cfg, comm=shared.for_rank(rank))
            outs[rank] = solver.step_owned(torch.from_numpy(moved[own]).to(dev),
                                           torch.from_numpy(system.charges[own]).to(dev),
                                           torch.from_numpy(own).to(dev), d_lam, d_nl, sites=tables,
                                           n_global=system.num_particles)
            torch.cuda.synchronize()
        except Exception as e:  # surfaced below
            errs.append(e)
            shared.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    n = system.num_particles
    forces = np.zeros((n, 3))
    count = np.zeros(n, int)
    for r, o in enumerate(outs):
        idx = o["owned"].cpu().numpy()
        a, b = ranges[r]
        assert np.all((lx_new[idx] >= a) & (lx_new[idx] < b)), "owned atoms lie in the rank's slab after the step"
        assert np.array_equal(o["owned_positions"].cpu().numpy(), moved[idx])
        forces[idx] = o["forces"].cpu().numpy()
        count[idx] += 1
    assert np.all(count == 1)
    assert abs(outs[0]["energy"] - e1) <= 1e-10 * abs(e1)
    assert relerr(forces, f1) <= 1e-10
    for o in outs:
        assert relerr(o["lambda_forces"].cpu().numpy(), lf1) <= 1e-10
