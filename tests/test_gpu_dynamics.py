"""Lambda dynamics on the device path (paper_2410_01754_b200/dynamics.py):
the reference's force-field identities (pkg/tests/test_dynamics.py:154-181:
frozen closed form = engine, HI and QI), the device-resident BAOAB loop
(run_trajectory_device) against the host loop at zero friction and
temperature (velocity Verlet: same trajectory), its reproducibility per
seed, and its Ornstein-Uhlenbeck noise variance kT/m."""

import numpy as np
import pytest
from numpy.testing import assert_allclose

pytestmark = pytest.mark.gpu

from paper_2410_01754_b200 import dynamics as dyn  # noqa: E402
from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig  # noqa: E402
from paper_2410_01754_b200.system import LambdaState, ParticleSystem, TitratableSite  # noqa: E402
from paper_2410_01754_b200.units import BOLTZMANN_KJ_PER_MOL_K  # noqa: E402


def small_system(seed, nforms=(2, 4), ns=4, n_bg=40, box=4.0):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0, box, (n_bg, 3))
    q = rng.uniform(-0.5, 0.5, n_bg)
    q -= q.mean()
    sites, allp = [], [pos]
    for s, nf in enumerate(nforms):
        c = rng.uniform(0, box, 3)
        allp.append((c + rng.uniform(-0.25, 0.25, (ns, 3))) % box)
        sites.append(TitratableSite(np.arange(n_bg + s * ns, n_bg + (s + 1) * ns), rng.uniform(-0.5, 0.5, (nf, ns))))
    system = ParticleSystem(box, np.vstack(allp), np.concatenate([q, np.zeros(len(nforms) * ns)]), sites)
    nl = [int(np.log2(nf)) for nf in nforms]
    lam = LambdaState(values=[rng.uniform(0.1, 0.9, k) for k in nl], velocities=[np.zeros(k) for k in nl],
                      masses=[5.0] * len(nforms))
    return system, lam


@pytest.mark.parametrize("images", ["full", "minimum"])
def test_frozen_field_matches_engine_field(images):
    system, _ = small_system(6)
    depth = 1 if images == "full" else 0
    cfg = SolverConfig(p=8, depth=depth, intra_site_images=images)
    frozen = dyn.FrozenLambdaForceField(system, config=cfg)
    engine = dyn.EngineLambdaForceField(system, config=cfg)
    for vals in ([np.array([0.3]), np.array([0.7, 0.2])], [np.array([0.9]), np.array([0.1, 0.5])]):
        ef, ff = frozen.lambda_forces(vals)
        ee, fe = engine.lambda_forces(vals)
        assert abs(ef - ee) < 1e-10 * max(1.0, abs(ee))
        for s in range(2):
            assert_allclose(ff[s], fe[s], rtol=0, atol=1e-10)


def test_frozen_field_qi_mode_matches_engine():
    system, _ = small_system(7, nforms=(2,))
    cfg = SolverConfig(p=6, depth=1)
    frozen = dyn.FrozenLambdaForceField(system, config=cfg, mode="qi")
    engine = dyn.EngineLambdaForceField(system, config=cfg, mode="qi")
    ef, ff = frozen.lambda_forces([np.array([0.37])])
    ee, fe = engine.lambda_forces([np.array([0.37])])
    assert abs(ef - ee) < 1e-10 * max(1.0, abs(ee))
    assert_allclose(ff[0], fe[0], rtol=0, atol=1e-10)


def test_device_trajectory_is_host_velocity_verlet():
    system, lam = small_system(8)
    lam.velocities = [np.full(len(v), 0.05) for v in lam.values]
    cfg = SolverConfig(p=8, depth=1)
    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    kw = dict(dt=0.002, temperature=0.0, friction=0.0, bias=dyn.BiasPotential(2.0), sample_every=4)
    host = dyn.run_trajectory(dyn.EngineLambdaForceField(system, solver=solver), lam.copy(), 40, **kw)
    ldev = lam.copy()
    dev = dyn.run_trajectory_device(system, ldev, 40, solver=solver, **kw)
    assert dev.lambdas.shape == host.lambdas.shape == (11, 3)
    assert_allclose(dev.times, host.times, rtol=0, atol=1e-15)
    assert_allclose(dev.lambdas, host.lambdas, rtol=0, atol=1e-10)
    assert_allclose(dev.velocities, host.velocities, rtol=0, atol=1e-9)
    assert_allclose(dev.forces, host.forces, rtol=1e-9, atol=1e-8)
    assert_allclose(dev.energies, host.energies, rtol=1e-11, atol=0)
    assert_allclose(np.concatenate(ldev.values), dev.lambdas[-1], rtol=0, atol=0)


def test_device_trajectory_reproducible_per_seed():
    system, lam = small_system(9)
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=6, depth=1))
    a = dyn.run_trajectory_device(system, lam.copy(), 20, solver=solver, seed=3)
    b = dyn.run_trajectory_device(system, lam.copy(), 20, solver=solver, seed=3)
    c = dyn.run_trajectory_device(system, lam.copy(), 20, solver=solver, seed=4)
    assert a.lambdas.tobytes() == b.lambdas.tobytes()
    assert a.velocities.tobytes() == b.velocities.tobytes()
    assert a.lambdas.tobytes() != c.lambdas.tobytes()
    assert np.all(np.isfinite(a.energies))


def test_device_noise_variance_is_kt_over_m():
    # friction * dt = 10: one step forgets the initial velocity; heavy masses
    # keep the force kicks (0.5 dt F / m) far below the thermal spread
    system, lam = small_system(10, nforms=(2,) * 256, ns=2, n_bg=64, box=8.0)
    m = 500.0
    lam.masses = [m] * 256
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=4, depth=1))
    t = dyn.run_trajectory_device(system, lam, 1, dt=0.002, temperature=300.0, friction=5000.0, solver=solver,
                                  bias=dyn.BiasPotential(0.0), seed=11)
    v = t.velocities[-1]
    sd = np.sqrt(BOLTZMANN_KJ_PER_MOL_K * 300.0 / m)
    assert abs(v.mean()) < 4 * sd / np.sqrt(v.size)
    assert abs(np.var(v) / sd ** 2 - 1.0) < 0.25


def test_frozen_field_trajectory_matches_reference_run():
    """The reference's run_trajectory over its FrozenLambdaForceField
    (dynamics.py:88-171, :214-285) on a small periodic system, HI mode, p=8,
    depth 1, thermostatted: this package's frozen field (device basis solve +
    device site Gram) under the host BAOAB reproduces every sample
    (tests/golden/dyn_frozen.npz)."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "dyn_frozen.npz"))
    sites = [TitratableSite(g["site0_idx"], g["site0_forms"]), TitratableSite(g["site1_idx"], g["site1_forms"])]
    system = ParticleSystem(float(g["box"]), g["positions"], g["charges"], sites)
    lam = LambdaState(values=[np.array([0.4]), np.array([0.7, 0.25])], velocities=[np.zeros(1), np.zeros(2)],
                      masses=[5.0, 5.0])
    field = dyn.FrozenLambdaForceField(system, config=SolverConfig(p=8, depth=1))
    t = dyn.run_trajectory(field, lam, 150, dt=0.002, temperature=300.0, friction=5.0,
                           rng=np.random.default_rng(21), sample_every=3)
    for key in ("times", "lambdas", "velocities"):
        assert_allclose(getattr(t, key), g[key], rtol=0, atol=1e-9, err_msg=key)
    assert_allclose(t.forces, g["forces"], rtol=0, atol=1e-9 * np.abs(g["forces"]).max())
    assert_allclose(t.energies, g["energies"], rtol=1e-11)
