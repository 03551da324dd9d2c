"""GPU HI parity: golden fixtures from the reference, and the reference's
HI identities restated (pkg/tests/test_corrections.py:145-312)."""

import itertools
import math

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import relerr

pytestmark = pytest.mark.gpu

from paper_2410_01754_b200 import (  # noqa: E402
    LambdaState, ParticleSystem, PeriodicSolver, SolverConfig, TitratableSite, assemble_lambda_forces,
    build_corrections, expand_weights, hi_energy_and_forces, scale_charges, weight_gradient_matrix)
from oracle import lfmm_oracle as orc  # noqa: E402


def system_from(g):
    off = g["site_atom_offsets"]
    nf = g["site_nforms"]
    forms = g["site_forms"]
    sites, fo = [], 0
    for s in range(len(nf)):
        ns = int(off[s + 1] - off[s])
        sites.append(TitratableSite(g["site_atoms"][off[s]:off[s + 1]], forms[fo:fo + nf[s] * ns].reshape(nf[s], ns)))
        fo += nf[s] * ns
    lam, lo = [], 0
    for n in g["n_lambda"]:
        lam.append(g["lambdas"][lo:lo + n])
        lo += n
    return ParticleSystem(float(g["box"]), g["positions"], g["charges"], sites), lam


def cfg_from(g, precision="double"):
    return SolverConfig(p=int(g["p"]), depth=int(g["depth"]), lattice_mode=str(g["lattice_mode"]),
                        shell_cap=int(g["shell_cap"]), dipole=bool(g["dipole"]), intra_site_images=str(g["intra"]),
                        precision=precision)


@pytest.mark.parametrize("name", ["hi_c1_water.npz", "hi_small_conv.npz", "hi_small_minimum.npz",
                                  "hi_small_nodip_shells.npz"])
@pytest.mark.parametrize("precision,tol", [("double", 1e-9), ("single", 1e-4)])
def test_hi_matches_reference_golden(golden, name, precision, tol):
    g = golden(name)
    system, lam = system_from(g)
    solver = PeriodicSolver(system.positions, system.box_length, cfg_from(g, precision))
    r = hi_energy_and_forces(system, lam, solver=solver)
    assert relerr(r.energy, g["hi_energy"]) <= tol
    assert relerr(np.concatenate(r.forces), g["hi_forces"]) <= tol
    assert relerr(r.solve.potentials, g["potentials"]) <= tol
    cs = r.corrections.sites
    ctol = 1e-11  # corrections are fp64 in both precisions
    assert relerr(np.concatenate([c.c_p2p for c in cs]), g["c_p2p"]) <= ctol
    if np.any(g["c_lattice"]):
        assert relerr(np.concatenate([c.c_lattice for c in cs]), g["c_lattice"]) <= ctol
    else:
        assert np.all(np.concatenate([c.c_lattice for c in cs]) == 0.0)
    if np.any(g["c_dipole"]):
        assert relerr(np.concatenate([c.c_dipole for c in cs]), g["c_dipole"]) <= ctol
    assert relerr(np.array([c.blend_energy for c in cs]), g["blend"]) <= ctol
    assert abs(r.corrections.energy_offset() - float(g["offset"])) <= ctol * max(1.0, abs(float(g["offset"])))
    rq = hi_energy_and_forces(system, lam, solver=solver, mode="qi")
    assert relerr(rq.energy, g["qi_energy"]) <= tol
    assert relerr(np.concatenate(rq.forces), g["qi_forces"]) <= tol
    assert rq.corrections is None


# ---- identities from pkg/tests/test_corrections.py ----
def make_system(n_bg=60, box=4.0, nforms=(2, 4), seed=77, compact=True):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0, box, (n_bg, 3))
    q = rng.uniform(-0.5, 0.5, n_bg)
    q -= q.mean()
    sites, all_pos, ns = [], [pos], 4
    for s, nf in enumerate(nforms):
        center = rng.uniform(0, box, 3)
        sp = center + rng.uniform(-0.25, 0.25, (ns, 3)) if compact else rng.uniform(0, box, (ns, 3))
        sp %= box
        all_pos.append(sp)
        sites.append(TitratableSite(np.arange(n_bg + s * ns, n_bg + (s + 1) * ns), rng.uniform(-0.5, 0.5, (nf, ns))))
    return ParticleSystem(box, np.vstack(all_pos), np.concatenate([q, np.zeros(len(nforms) * ns)]), sites)


def end_state_charges(system, assignment):
    q = system.charges.copy()
    for site, rho in zip(system.sites, assignment):
        q[site.particle_indices] = site.form_charges[rho]
    return q


def blend_reference(system, lam_values, solver):
    nfs = [s.num_forms for s in system.sites]
    assigns = list(itertools.product(*[range(nf) for nf in nfs]))
    cols = np.stack([end_state_charges(system, a) for a in assigns], axis=1)
    energies = np.asarray(solver.solve(cols).energy)
    tilde = [expand_weights(v) for v in lam_values]
    grads = [weight_gradient_matrix(v) for v in lam_values]
    w = np.ones(len(assigns))
    for k, a in enumerate(assigns):
        for s, rho in enumerate(a):
            w[k] *= tilde[s].values[rho]
    e_blend = math.fsum((w * energies).tolist())
    forces = []
    for s, lams in enumerate(lam_values):
        gvec = np.zeros(len(lams))
        for i in range(len(lams)):
            acc = []
            for k, a in enumerate(assigns):
                wpart = 1.0
                for s2, rho2 in enumerate(a):
                    if s2 != s:
                        wpart *= tilde[s2].values[rho2]
                acc.append(wpart * grads[s][i, a[s]] * energies[k])
            gvec[i] = math.fsum(acc)
        forces.append(-gvec)
    return e_blend, forces


@pytest.mark.parametrize("p", [2, 8, 16])
def test_identity_depth0_machine_exact(p):
    system = make_system()
    lam = [np.array([0.345]), np.array([0.345, 0.721])]
    cfg = SolverConfig(p=p, depth=0, lattice_mode="shells", shell_cap=4, dipole=True)
    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    r = hi_energy_and_forces(system, lam, solver=solver)
    eb, fb = blend_reference(system, lam, solver)
    assert abs(r.energy - eb) / abs(eb) < 1e-12
    assert max(relerr(r.forces[s], fb[s]) for s in range(2)) < 5e-13


def test_identity_depth0_converged_lattice():
    system = make_system(seed=5)
    lam = [np.array([0.42]), np.array([0.1, 0.9])]
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=8, depth=0))
    r = hi_energy_and_forces(system, lam, solver=solver)
    eb, fb = blend_reference(system, lam, solver)
    assert abs(r.energy - eb) / abs(eb) < 1e-12
    assert max(relerr(r.forces[s], fb[s]) for s in range(2)) < 5e-13


@pytest.mark.parametrize("dipole", [True, False])
def test_vertex_consistency(dipole):
    system = make_system(seed=9)
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=6, depth=1, dipole=dipole))
    for vertex in ((np.array([1.0]), np.array([0.0, 1.0])), (np.array([0.0]), np.array([1.0, 1.0]))):
        r = hi_energy_and_forces(system, vertex, solver=solver)
        assign = tuple(sum(int(round(l)) << i for i, l in enumerate(lams)) for lams in vertex)
        ev = float(solver.solve(end_state_charges(system, assign)).energy)
        assert abs(r.energy - ev) / max(abs(ev), 1.0) < 1e-13


def test_assembled_forces_match_finite_difference():
    system = make_system(seed=13)
    lam = [np.array([0.345]), np.array([0.345, 0.721])]
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=1))
    r = hi_energy_and_forces(system, lam, solver=solver)
    h = 1e-5
    for s in range(2):
        for i in range(len(lam[s])):
            hi = [v.copy() for v in lam]
            lo = [v.copy() for v in lam]
            hi[s][i] += h
            lo[s][i] -= h
            fd = -(hi_energy_and_forces(system, hi, solver=solver).energy
                   - hi_energy_and_forces(system, lo, solver=solver).energy) / (2 * h)
            assert abs(fd - r.forces[s][i]) < 1e-7


def test_qi_energy_is_blended_charge_solve():
    system = make_system(seed=21)
    lam = [np.array([0.6]), np.array([0.3, 0.2])]
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=8, depth=1))
    rq = hi_energy_and_forces(system, lam, solver=solver, mode="qi")
    qt = scale_charges(system, [expand_weights(v) for v in lam])
    assert abs(rq.energy - float(solver.solve(qt).energy)) < 1e-12
    assert rq.corrections is None


def k_factor(pos, dq, box):
    disp = pos[:, None, :] - pos[None, :, :]
    disp = disp - box * np.round(disp / box)
    r = np.sqrt((disp * disp).sum(-1))
    np.fill_diagonal(r, np.inf)
    return math.fsum(((dq[:, None] * dq[None, :]) / r).ravel().tolist())


def test_hi_qi_gap_is_linear_for_two_form_sites():
    system = make_system(nforms=(2, 2), seed=31)
    solver = PeriodicSolver(system.positions, system.box_length,
                            SolverConfig(p=8, depth=1, intra_site_images="minimum"))
    ks = [k_factor(system.positions[s.particle_indices], s.form_charges[1] - s.form_charges[0], system.box_length)
          for s in system.sites]
    for lam_a, lam_b in (([0.3], [0.6]), ([0.9], [0.1])):
        lam = [np.array(lam_a), np.array(lam_b)]
        rh = hi_energy_and_forces(system, lam, solver=solver, mode="hi")
        rq = hi_energy_and_forces(system, lam, solver=solver, mode="qi")
        for s, lv in enumerate(lam):
            assert abs((rh.forces[s][0] - rq.forces[s][0]) - (lv[0] - 0.5) * ks[s]) < 1e-9 * max(abs(ks[s]), 1.0)


def test_build_corrections_minimum_mode_drops_far_terms():
    system = make_system(seed=41)
    lam = [np.array([0.5]), np.array([0.5, 0.5])]
    solver = PeriodicSolver(system.positions, system.box_length,
                            SolverConfig(p=6, depth=0, intra_site_images="minimum"))
    cs = build_corrections(system, lam, solver)
    for site in cs.sites:
        assert np.all(site.c_lattice == 0.0)
        assert np.all(site.c_dipole == 0.0)


def test_stale_corrections_rejected():
    system = make_system(seed=43)
    lam = [np.array([0.5]), np.array([0.25, 0.75])]
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=6, depth=0))
    cs = build_corrections(system, lam, solver)
    res = solver.solve(scale_charges(system, [expand_weights(v) for v in lam]))
    with pytest.raises(ValueError, match="different lambda"):
        assemble_lambda_forces(system, [np.array([0.6]), np.array([0.25, 0.75])], cs, res.potentials)


def test_split_api_matches_fused():
    system = make_system(seed=44)
    lam = [np.array([0.3]), np.array([0.25, 0.75])]
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=8, depth=1))
    fused = hi_energy_and_forces(system, lam, solver=solver)
    cs = build_corrections(system, lam, solver)
    res = solver.solve(scale_charges(system, [expand_weights(v) for v in lam]))
    f = assemble_lambda_forces(system, lam, cs, res.potentials)
    for s in range(2):
        assert_allclose(f[s], fused.forces[s], rtol=1e-12, atol=1e-12)
    assert abs(float(res.energy) + cs.energy_offset() - fused.energy) < 1e-12 * abs(fused.energy)


def test_lambda_state_input_accepted():
    system = make_system(seed=47)
    state = LambdaState(values=[[0.3], [0.6, 0.1]], velocities=[[0.0], [0.0, 0.0]], masses=[5.0, 5.0])
    cfg = SolverConfig(p=6, depth=0)
    a = hi_energy_and_forces(system, state, config=cfg)
    b = hi_energy_and_forces(system, [np.array([0.3]), np.array([0.6, 0.1])], config=cfg)
    assert a.energy == b.energy
    for s in range(2):
        assert_allclose(a.forces[s], b.forces[s], rtol=0, atol=0)


def test_bad_mode_and_mismatched_lambdas():
    system = make_system(seed=48)
    with pytest.raises(ValueError, match="unknown mode"):
        hi_energy_and_forces(system, [[0.5], [0.5, 0.5]], config=SolverConfig(p=4, depth=0), mode="xx")
    with pytest.raises(ValueError, match="weights, site has"):
        hi_energy_and_forces(system, [[0.5, 0.5], [0.5, 0.5]], config=SolverConfig(p=4, depth=0))


def test_hi_oracle_c1_fp32_and_fp64(golden):
    """C1 water box: GPU vs the CPU oracle (itself pinned to the reference)."""
    g = golden("hi_c1_water.npz")
    system, lam = system_from(g)
    sites = [(s.particle_indices, s.form_charges) for s in system.sites]
    cfg = dict(p=8, depth=3, lattice_mode="converged", shell_cap=8, dipole=True, periodic_near=True,
               intra_site_images="full")
    ref = orc.hi(system.positions, system.charges, system.box_length, sites, lam, cfg)
    for precision, tol in (("double", 1e-9), ("single", 1e-4)):
        solver = PeriodicSolver(system.positions, system.box_length, cfg_from(g, precision))
        r = hi_energy_and_forces(system, lam, solver=solver)
        assert relerr(r.energy, ref["energy"]) <= tol
        assert relerr(np.concatenate(r.forces), np.concatenate(ref["forces"])) <= tol
