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
                                           ("LFMM_FAR=serial", "single"), ("LFMM_M2L64=gather", "double")])
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


def test_far_serial_matches_overlapped(monkeypatch):
    """far_overlapped() runs the small levels on a second stream; the only
    arithmetic difference is that their M2M reads level ls with the exact
    box charges already applied (serial: applied after every M2M), an fp32
    rounding-level change (depth 5 so the split is active).  Each order is
    bit-reproducible on its own (test_gpu_solve reruns)."""
    system, lam, _ = generate_water_box(200_000, 16, seed=3)
    cfg = SolverConfig(p=10, depth=5, precision="single")
    a = PeriodicSolver(system.positions, system.box_length, cfg).solve(system.charges)
    monkeypatch.setenv("LFMM_FAR", "serial")
    b = PeriodicSolver(system.positions, system.box_length, cfg).solve(system.charges)
    assert relerr(b.potentials, a.potentials) <= 2e-6


def test_non_finite_result_raises_numerical_failure():
    """Status 3 -> NumericalFailure (the reference CLI's exit-2 class,
    cli.py:24-25): a NaN charge poisons the energies."""
    system, lam, _ = generate_water_box(3000, 4, seed=0)
    q = np.array(system.charges)
    q[17] = np.nan
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=6, depth=2))
    with pytest.raises(NumericalFailure, match="non-finite"):
        solver.solve(q)
