"""The A/B kernel switches the plan reads at creation (lfmm_plan_create):
each alternative path is checked against the pinned oracle on the C1 water
box, so no selectable code path goes untested; plus the NumericalFailure
status (3) of non-finite results."""

import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu

from oracle import lfmm_oracle as orc  # noqa: E402
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig, hi_energy_and_forces  # noqa: E402
from paper_2410_01754_b200._native import NumericalFailure  # noqa: E402
from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

_ref = {}


def c1():
    if not _ref:
        system, lam, _ = generate_water_box(3000, 4, seed=0)
        sites = [(s.particle_indices, s.form_charges) for s in system.sites]
        cfg = orc.default_config(p=10, depth=3)
        ref = orc.hi(system.positions, system.charges, system.box_length, sites, lam.values, cfg)
        fq = orc.solve(system.positions, ref["q_tilde"], system.box_length, cfg, forces=True)["forces"]
        _ref.update(system=system, lam=lam, ref=ref, fq=fq)
    return _ref


@pytest.mark.parametrize("env,precision", [("LFMM_M2L=simt", "single"), ("LFMM_P2P=scalar", "single"),
                                           ("LFMM_P2P=plain", "single"), ("LFMM_M2L64=gather", "double"),
                                           ("LFMM_GRAPH=0", "single"), ("LFMM_TRANSLATE=simt", "single")])
def test_switch_matches_oracle(env, precision, monkeypatch):
    d = c1()
    name, val = env.split("=")
    monkeypatch.setenv(name, val)
    system, lam, ref = d["system"], d["lam"], d["ref"]
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=3, precision=precision))
    monkeypatch.delenv(name)
    r = hi_energy_and_forces(system, lam.values, solver=solver, mode="qi", spatial_forces=True)
    tol = 1e-4 if precision == "single" else 1e-9
    assert relerr(r.solve.potentials, ref["solve"]["potentials"]) <= tol
    assert relerr(r.energy, ref["energy"] - sum(ref["offset"])) <= tol
    assert relerr(r.spatial_forces, d["fq"]) <= tol


def test_preemptible_near_field_and_step_graph_are_bit_identical(monkeypatch):
    """The default fp32 near field runs as three persistent launches that
    share one leaf counter (lfmm_api.cu solve_column: beside the far-field
    chains, yielding to the M2L); every leaf is computed by one warp with the
    same arithmetic whichever launch takes it, so potentials and forces equal
    the single-launch schedule (LFMM_P2P=plain) bit for bit (depth 5: the
    schedule is active); the step replayed from its CUDA graph equals the
    uncaptured step (LFMM_GRAPH=0) bit for bit."""
    import torch

    from paper_2410_01754_b200 import _native
    from paper_2410_01754_b200.system import lambda_table, site_tables

    system, lam, _ = generate_water_box(200_000, 16, seed=3)
    cfg = SolverConfig(p=10, depth=5, precision="single")
    outs = []
    for plain in (False, True, "nograph"):
        if plain is True:
            monkeypatch.setenv("LFMM_P2P", "plain")
        if plain == "nograph":
            monkeypatch.delenv("LFMM_P2P")
            monkeypatch.setenv("LFMM_GRAPH", "0")
        solver = PeriodicSolver(system.positions, system.box_length, cfg)
        plan = solver.plan
        plan.set_sites(*site_tables(system))
        lt, nl = lambda_table(system, lam.values)
        dev = torch.device("cuda", 0)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        e = torch.empty(1, dtype=torch.float64, device=dev)
        f = torch.empty((system.num_particles, 3), dtype=torch.float64, device=dev)
        lf = torch.empty((len(system.sites), 4), dtype=torch.float64, device=dev)
        args = (d(system.positions), d(system.charges), d(lt), d(nl))
        for _ in range(3):  # warm-up, capture + replay, replay (the step graph, unless LFMM_GRAPH=0)
            plan.step(*args, mode=_native.MODE_HI, on_device=True, energy=e, forces=f, lambda_forces=lf)
        torch.cuda.synchronize()
        outs.append((e.cpu().numpy(), f.cpu().numpy(), lf.cpu().numpy()))
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert a.tobytes() == b.tobytes()


def test_non_finite_result_raises_numerical_failure():
    """Status 3 -> NumericalFailure (the reference CLI's exit-2 class,
    cli.py:24-25): a NaN charge poisons the energies."""
    system, lam, _ = generate_water_box(3000, 4, seed=0)
    q = np.array(system.charges)
    q[17] = np.nan
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=6, depth=2))
    with pytest.raises(NumericalFailure, match="non-finite"):
        solver.solve(q)


def test_step_graph_follows_new_site_tables():
    """A captured step bakes in sizes (site count, grids): replacing the site
    tables with fewer sites between calls must re-capture, so the step equals
    a fresh plan's uncaptured step."""
    import torch

    from paper_2410_01754_b200 import _native
    from paper_2410_01754_b200.system import ParticleSystem, lambda_table, site_tables

    system, lam, _ = generate_water_box(20_000, 8, seed=5)
    fewer = ParticleSystem(system.box_length, system.positions, system.charges, system.sites[:3])
    cfg = SolverConfig(p=8, depth=3, precision="single")
    dev = torch.device("cuda", 0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731

    def run(plan, sysm, lam_values, reps):
        lt, nl = lambda_table(sysm, lam_values)
        e = torch.empty(1, dtype=torch.float64, device=dev)
        f = torch.empty((sysm.num_particles, 3), dtype=torch.float64, device=dev)
        lf = torch.empty((8, 4), dtype=torch.float64, device=dev)
        args = (d(sysm.positions), d(sysm.charges), d(lt), d(nl))
        for _ in range(reps):
            plan.step(*args, mode=_native.MODE_HI, on_device=True, energy=e, forces=f, lambda_forces=lf)
        torch.cuda.synchronize()
        return float(e.cpu()[0]), f.cpu().numpy(), lf.cpu().numpy()[: len(sysm.sites)]

    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    solver.plan.set_sites(*site_tables(system))
    run(solver.plan, system, lam.values, 3)  # captured with 8 sites
    solver.plan.set_sites(*site_tables(fewer))
    got = run(solver.plan, fewer, lam.values[:3], 3)
    fresh = PeriodicSolver(system.positions, system.box_length, cfg)
    fresh.plan.set_sites(*site_tables(fewer))
    want = run(fresh.plan, fewer, lam.values[:3], 1)
    assert got[0] == want[0]
    assert got[1].tobytes() == want[1].tobytes() and got[2].tobytes() == want[2].tobytes()
