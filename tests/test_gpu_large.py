"""GPU parity at the benchmark sizes.

C2 (~100k atoms, 64 sites, p=10, depth 4): the fp64 device path against the
CPU oracle for the whole solve (potentials, near/far pieces, energies, forces)
and the HI lambda forces; the fp32 path (tensor-core M2L) against the fp64
device path.  C3 (~1M atoms, 512 sites, p=10, depth 5): fp32 against fp64 on
the device, and the oracle on a sample of leaves for the near field.
Tolerances are the north_star's: 1e-6 in fp64, 1e-4 in fp32 (max-normalised,
the reference's metric, bench.py:46-52)."""

import numpy as np
import pytest

from conftest import relerr

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from paper_2410_01754_b200 import PeriodicSolver, SolverConfig, hi_energy_and_forces  # noqa: E402
from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402
from oracle import lfmm_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def c2():
    system, lam, _ = generate_water_box(100_000, 64, seed=3)
    return system, lam


@pytest.fixture(scope="module")
def c3():
    system, lam, _ = generate_water_box(1_000_000, 512, seed=4)
    return system, lam


def _solve(system, p, depth, precision, forces=True):
    s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=p, depth=depth, precision=precision))
    r = s.solve(system.charges)
    f = s.spatial_forces(system.charges) if forces else None
    return s, r, f


def test_c2_fp64_matches_oracle(c2):
    system, lam = c2
    _, r, f = _solve(system, 10, 4, "double")
    ref = orc.solve(system.positions, system.charges, system.box_length, orc.default_config(p=10, depth=4),
                    forces=True)
    assert relerr(r.potentials, ref["potentials"]) <= 1e-6
    assert relerr(r.near_potentials, ref["near"]) <= 1e-6
    assert relerr(r.far_potentials, ref["far"]) <= 1e-6
    assert relerr(r.energy, ref["energy"]) <= 1e-6
    assert relerr(f, ref["forces"]) <= 1e-6


@pytest.mark.parametrize("depth", [4, 5])
def test_c2_fp32_matches_fp64(c2, depth):
    system, lam = c2
    _, r64, f64 = _solve(system, 10, depth, "double")
    _, r32, f32 = _solve(system, 10, depth, "single")
    for a, b in ((r32.potentials, r64.potentials), (r32.near_potentials, r64.near_potentials),
                 (r32.far_potentials, r64.far_potentials), (r32.dipole_potentials, r64.dipole_potentials)):
        assert relerr(a, b) <= 1e-4
    for k in ("energy", "near_energy", "far_energy", "dipole_energy"):
        assert relerr(getattr(r32, k), getattr(r64, k)) <= 1e-4, k
    assert relerr(f32, f64) <= 1e-4
    assert relerr(r32.root_multipole, r64.root_multipole) <= 1e-4


def test_c2_hi_fp32_matches_fp64(c2):
    system, lam = c2
    out = {}
    for prec in ("double", "single"):
        s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=4, precision=prec))
        out[prec] = hi_energy_and_forces(system, lam.values, solver=s)
    assert relerr(out["single"].energy, out["double"].energy) <= 1e-4
    assert relerr(np.concatenate(out["single"].forces), np.concatenate(out["double"].forces)) <= 1e-4


def test_c3_fp32_matches_fp64(c3):
    system, lam = c3
    _, r64, f64 = _solve(system, 10, 5, "double")
    _, r32, f32 = _solve(system, 10, 5, "single")
    err = {
        "potentials": relerr(r32.potentials, r64.potentials),
        "far": relerr(r32.far_potentials, r64.far_potentials),
        "near": relerr(r32.near_potentials, r64.near_potentials),
        "forces": relerr(f32, f64),
        "energy": relerr(r32.energy, r64.energy),
    }
    print("C3 fp32 vs fp64:", err)
    assert max(err.values()) <= 1e-4, err


def test_c3_fp64_near_field_matches_oracle_sample(c3):
    system, lam = c3
    s, r64, _ = _solve(system, 10, 5, "double", forces=False)
    tree = orc.build_tree(orc.wrap(system.positions, system.box_length), system.box_length, 5)
    q = system.charges[tree["perm"]][:, None]
    leaves = np.arange(0, 2 ** 15, 97)
    v, _ = orc.near_field(tree, q, leaves=leaves)
    idx = np.concatenate([np.arange(tree["leaf_start"][b], tree["leaf_start"][b + 1]) for b in leaves])
    ref = v[idx, 0]
    got = r64.near_potentials[tree["perm"][idx]]
    assert relerr(got, ref) <= 1e-9


def test_depth6_fp32_matches_fp64():
    """Depth 6 (C5's tree; level-6 halo windows run the 10-stage A ring of
    k_m2l_halo): the fp32 step against the fp64 device solve."""
    system, _, _ = generate_water_box(300_000, 0, seed=6)
    _, r64, f64 = _solve(system, 10, 6, "double")
    _, r32, f32 = _solve(system, 10, 6, "single")
    assert relerr(r32.potentials, r64.potentials) <= 1e-4
    assert relerr(r32.far_potentials, r64.far_potentials) <= 1e-4
    assert relerr(r32.energy, r64.energy) <= 1e-4
    assert relerr(f32, f64) <= 1e-4
