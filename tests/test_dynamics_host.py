"""Host pieces of the lambda dynamics (paper_2410_01754_b200/dynamics.py),
restating the reference's own tests (pkg/tests/test_dynamics.py:12-47,
49-74, 77-95, 98-109, 184-189): bias/wall shapes and FD forces, BAOAB at
zero friction and temperature = velocity Verlet, equipartition, transition
counting, replica streams.  No GPU: the force fields here are analytic."""

import numpy as np
import pytest
from numpy.testing import assert_allclose

from paper_2410_01754_b200 import dynamics as dyn
from paper_2410_01754_b200.system import LambdaState
from paper_2410_01754_b200.units import BOLTZMANN_KJ_PER_MOL_K, COULOMB_KJ_PER_MOL


def test_bias_is_midpoint_barrier():
    bias = dyn.BiasPotential(height=5.0)
    assert bias.energy(np.array([0.5])) == 5.0
    assert bias.energy(np.array([0.0])) == 0.0
    assert bias.energy(np.array([1.0])) == 0.0
    assert bias.force(np.array([0.4]))[0] < 0
    assert bias.force(np.array([0.6]))[0] > 0


def test_bias_and_wall_forces_match_fd():
    bias = dyn.BiasPotential(height=3.0)
    h = 1e-7
    for x in (0.17, 0.5, 0.83, 1.05):
        fd = -(bias.energy(np.array([x + h])) - bias.energy(np.array([x - h]))) / (2 * h)
        assert_allclose(bias.force(np.array([x]))[0], fd, rtol=0, atol=1e-6)
    for x in (-0.25, -0.11, 0.5, 1.14, 1.3):
        fd = -(dyn.wall_energy(np.array([x + h])) - dyn.wall_energy(np.array([x - h]))) / (2 * h)
        assert_allclose(dyn.wall_force(np.array([x]))[0], fd, rtol=1e-6, atol=1e-4)
    assert dyn.wall_energy(np.array([0.0])) == 0.0
    assert dyn.wall_force(np.array([0.5]))[0] == 0.0


class ConstField:
    def __init__(self, f_internal):
        self.f = f_internal

    def lambda_forces(self, lam_values):
        return 0.0, [np.full(len(v), self.f) for v in lam_values]


class SpringField:
    def lambda_forces(self, lam_values):
        k_int = 100.0 / COULOMB_KJ_PER_MOL
        return 0.0, [-k_int * (v - 0.5) for v in lam_values]


def test_zero_friction_zero_temperature_is_velocity_verlet():
    f_int = 2.5e-3
    f_kj = f_int * COULOMB_KJ_PER_MOL
    m = 5.0
    lam = LambdaState(values=[np.array([0.3])], velocities=[np.array([0.04])], masses=[m])
    traj = dyn.run_trajectory(ConstField(f_int), lam, 100, dt=0.002, temperature=0.0, friction=0.0,
                              bias=dyn.BiasPotential(0.0))
    t = traj.times[-1]
    assert abs(traj.lambdas[-1, 0] - (0.3 + 0.04 * t + 0.5 * (f_kj / m) * t * t)) < 1e-10
    assert abs(traj.velocities[-1, 0] - (0.04 + (f_kj / m) * t)) < 1e-12
    assert_allclose(lam.values[0], traj.lambdas[-1], rtol=0, atol=0)  # state written back


@pytest.mark.slow
def test_thermostat_equipartition():
    m = 5.0
    lam = LambdaState(values=[np.array([0.5])], velocities=[np.array([0.0])], masses=[m])
    traj = dyn.run_trajectory(SpringField(), lam, 300000, dt=0.002, temperature=300.0, friction=5.0,
                              bias=dyn.BiasPotential(0.0), rng=np.random.default_rng(42))
    v = traj.velocities[10000:, 0]
    assert abs(np.var(v) * m / (BOLTZMANN_KJ_PER_MOL_K * 300.0) - 1.0) < 0.05


def test_transition_counting_pinned():
    n, _ = dyn.count_transitions(np.linspace(0, 1, 101))
    assert n == 1
    square = np.concatenate([np.full(10, i % 2) for i in range(7)])
    n, flips = dyn.count_transitions(square)
    assert n == 6 and len(flips) == 6
    n, _ = dyn.count_transitions(np.array([0.0, 0.3, 0.7, 0.3, 0.7, 0.3, 0.0, 0.9]))
    assert n == 1


def test_trajectory_sampling_and_determinism():
    lam = LambdaState(values=[np.array([0.3]), np.array([0.6, 0.2])], velocities=[np.zeros(1), np.zeros(2)],
                      masses=[5.0, 5.0])
    a = dyn.run_trajectory(SpringField(), lam.copy(), 50, rng=np.random.default_rng(9), sample_every=5)
    b = dyn.run_trajectory(SpringField(), lam.copy(), 50, rng=np.random.default_rng(9), sample_every=5)
    assert a.lambdas.shape == (11, 3)
    assert_allclose(np.diff(a.times), 0.01, rtol=0, atol=1e-15)
    assert a.lambdas.tobytes() == b.lambdas.tobytes()
    assert [r.slot for r in a.transitions()] == [0, 0, 1]


def test_replica_rng_streams_differ_and_reproduce():
    a = dyn.replica_rng(7, 0).standard_normal(4)
    assert_allclose(a, dyn.replica_rng(7, 0).standard_normal(4), rtol=0, atol=0)
    assert not np.allclose(a, dyn.replica_rng(7, 1).standard_normal(4))


class CoupledSprings:
    """tests/golden/make_golden_dynamics.py CoupledSprings (same formula)."""

    def lambda_forces(self, lam_values):
        flat = np.concatenate([np.asarray(v, float) for v in lam_values])
        k, g = 80.0 / COULOMB_KJ_PER_MOL, 15.0 / COULOMB_KJ_PER_MOL
        centre = np.linspace(0.35, 0.65, flat.size)
        f = -k * (flat - centre) - g * (flat.sum() - flat)
        e = 0.5 * k * float(((flat - centre) ** 2).sum())
        out, o = [], 0
        for v in lam_values:
            out.append(f[o:o + len(v)])
            o += len(v)
        return e, out


def test_thermostatted_trajectory_matches_reference_run():
    """The reference's own run_trajectory (dynamics.py:214-285) on a coupled
    spring field, thermostatted, two sites, sample_every=7: same samples to
    round-off, same final state (tests/golden/dyn_spring.npz)."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "dyn_spring.npz"))
    lam = LambdaState(values=[np.array([0.3]), np.array([0.6, 0.2])], velocities=[np.array([0.1]), np.zeros(2)],
                      masses=[5.0, 3.0])
    t = dyn.run_trajectory(CoupledSprings(), lam, 400, dt=0.002, temperature=300.0, friction=5.0,
                           bias=dyn.BiasPotential(4.0), rng=np.random.default_rng(9), sample_every=7)
    for key in ("times", "lambdas", "velocities", "forces", "energies"):
        assert_allclose(getattr(t, key), g[key], rtol=1e-12, atol=1e-12, err_msg=key)
    assert_allclose(np.concatenate(lam.values), g["final_values"], rtol=1e-12, atol=1e-12)
    assert_allclose(np.concatenate(lam.velocities), g["final_velocities"], rtol=1e-12, atol=1e-12)
