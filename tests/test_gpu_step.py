"""The benchmarked step itself (lfmm_step, bench.py step_dev) against the
reference and the pinned oracle.

bench.py times ``plan.step(d_pos, d_q, d_lam, d_nl, MODE_HI, on_device=True)``:
device inputs, positions passed every step (per-step tree rebuild), the HI
corrections issued on a side stream before the tree, then one tail kernel
(k_step_tail) that rebuilds the site potentials from the canonical pieces,
forms the lambda forces, adds the HI site-atom spatial forces into the force
rows and writes the step energy.  These tests run exactly that call and compare

* energy with the reference's hi_energy_and_forces(...).energy
  (corrections.py:252-274),
* lambda forces with its InterpolationResult.forces,
* forces with spatial_forces(q~) (solver.py:407-427) plus, on site atoms,
  -grad Delta E_site (reference central differences of its own per-site
  correction pieces, tests/golden/ref_site_forces.npz),
* the rebuilt tree with the reference's build_octree (octree.py:114-163)
  by sha256 of perm and leaf_start,

at C1 (full arrays, oracle), C2 and C3 (reference fixtures).  Tolerances are
the north_star's: 1e-6 (fp64) and 1e-4 (fp32), max-normalised
(bench.py:46-52)."""

import copy
import hashlib
import os

import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu

from oracle import lfmm_oracle as orc  # noqa: E402
from paper_2410_01754_b200 import _native  # noqa: E402
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig, hi_energy_and_forces  # noqa: E402
from paper_2410_01754_b200.system import lambda_table, site_tables  # noqa: E402
from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"double": 1e-6, "single": 1e-4}
_systems = {}


def water(n, ns, seed):
    key = (n, ns, seed)
    if key not in _systems:
        _systems[key] = generate_water_box(n, ns, seed=seed)[:2]
    return _systems[key]


def checksum(system):
    return np.array([system.positions.sum(), (system.positions ** 2).sum(), system.charges.sum(),
                     np.abs(system.charges).sum(), float(system.num_particles)])


class Stepper:
    """bench.py's device-resident step (run_ours.step_dev), same call."""

    def __init__(self, system, lam_values, cfg):
        import torch

        self.torch = torch
        dev = torch.device("cuda", 0)
        self.solver = PeriodicSolver(system.positions, system.box_length, cfg)
        self.plan = self.solver.plan
        self.plan.set_sites(*site_tables(system))
        lam, nl = lambda_table(system, lam_values)
        self.stream = torch.cuda.Stream(device=dev)
        self.plan.set_stream(self.stream.cuda_stream)
        n, s = system.num_particles, len(system.sites)
        self.n, self.s = n, s
        self.d_q = torch.from_numpy(np.ascontiguousarray(system.charges)).to(dev)
        self.d_lam = torch.from_numpy(np.ascontiguousarray(lam)).to(dev)
        self.d_nl = torch.from_numpy(np.ascontiguousarray(nl)).to(dev)
        self.d_e = torch.empty(1, dtype=torch.float64, device=dev)
        self.d_f = torch.empty((n, 3), dtype=torch.float64, device=dev)
        self.d_lf = torch.empty((max(s, 1), 4), dtype=torch.float64, device=dev)
        self.dev = dev

    def step(self, positions, mode=_native.MODE_HI):
        torch = self.torch
        d_pos = torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float64)).to(self.dev)
        torch.cuda.synchronize()
        self.plan.step(d_pos, self.d_q, self.d_lam, self.d_nl, mode=mode, plain=False, on_device=True,
                       energy=self.d_e, forces=self.d_f, lambda_forces=self.d_lf)
        self.stream.synchronize()
        return (float(self.d_e.cpu()[0]), self.d_f.cpu().numpy().copy(),
                self.d_lf.cpu().numpy()[: self.s].copy())

    def tree_hashes(self):
        perm, _, _, start, _ = self.plan.export_tree()
        return (hashlib.sha256(perm.astype(np.int64).tobytes()).hexdigest(),
                hashlib.sha256(start.astype(np.int64).tobytes()).hexdigest(), perm)


def lambda_rows(system, lam_values, lf):
    nl = [site.num_lambda for site in system.sites]
    return np.concatenate([lf[i, : nl[i]] for i in range(len(nl))]) if nl else np.zeros(0)


def site_force_fixture(tag):
    g = np.load(os.path.join(GOLDEN, "ref_site_forces_c4.npz" if tag == "c4" else "ref_site_forces.npz"))
    return g[tag + "_idx"], g[tag + "_dforce"], g[tag + "_checksum"]


# ------------------------------------------------------------ C1, oracle ----
@pytest.mark.parametrize("precision", ["double", "single"])
def test_step_c1_full_arrays(precision):
    """C1 water box (3k atoms, 4 sites, p=8, d=3): every force row, the
    energy and the lambda forces of the benchmarked step against the oracle
    (pinned to the reference) plus the reference's site-force corrections."""
    system, lam = water(3000, 4, 0)
    cfg = SolverConfig(p=8, depth=3, precision=precision)
    ocfg = orc.default_config(p=8, depth=3)
    sites = [(s.particle_indices, s.form_charges) for s in system.sites]
    ref = orc.hi(system.positions, system.charges, system.box_length, sites, lam.values, ocfg)
    fq = orc.solve(system.positions, ref["q_tilde"], system.box_length, ocfg, forces=True)["forces"]
    idx, dforce, ck = site_force_fixture("c1")
    np.testing.assert_allclose(ck, checksum(system), rtol=1e-13)
    f_ref = fq.copy()
    f_ref[idx] += dforce
    st = Stepper(system, lam.values, cfg)
    for _ in range(2):  # second call: the steady state bench.py times
        e, f, lf = st.step(system.positions)
    tol = TOL[precision]
    assert relerr(e, ref["energy"]) <= tol
    assert relerr(lambda_rows(system, lam.values, lf), np.concatenate(ref["forces"])) <= tol
    assert relerr(f, f_ref) <= tol
    # the site-atom correction is really there: QI-only forces differ from it
    assert relerr(f[idx], fq[idx]) > 10 * tol or precision == "single"


def test_step_qi_mode_forces_are_charge_scaled():
    """QI mode: E = E_solve(q~), forces = spatial_forces(q~) everywhere (no
    site term; corrections.py:268-270)."""
    system, lam = water(3000, 4, 0)
    cfg = SolverConfig(p=8, depth=3)
    ocfg = orc.default_config(p=8, depth=3)
    sites = [(s.particle_indices, s.form_charges) for s in system.sites]
    ref = orc.hi(system.positions, system.charges, system.box_length, sites, lam.values, ocfg, mode="qi")
    fq = orc.solve(system.positions, ref["q_tilde"], system.box_length, ocfg, forces=True)["forces"]
    st = Stepper(system, lam.values, cfg)
    e, f, lf = st.step(system.positions, mode=_native.MODE_QI)
    assert relerr(e, ref["energy"]) <= 1e-9
    assert relerr(f, fq) <= 1e-9
    assert relerr(lambda_rows(system, lam.values, lf), np.concatenate(ref["forces"])) <= 1e-9


# --------------------------------------------------- C2 / C3, reference ----
@pytest.mark.slow
@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("case", ["c2", "c3", "c4", "c3d6"])
def test_step_matches_reference(case, precision):
    """C2 (100k, 64 sites, d=4), C3 (1M, 512 sites, d=5), C4 (1M, 4096
    sites, d=5: the HI site-count stress box) and the C3 box at the
    reference's depth cap d=6 (solver.py:62-64)."""
    name = {"c2": "ref_c2_d4.npz", "c3": "ref_c3_d5.npz", "c4": "ref_c4_d5.npz", "c3d6": "ref_c3_d6.npz"}[case]
    g = np.load(os.path.join(GOLDEN, name))
    system, lam = water(int(g["n_atoms"]), int(g["n_sites"]), int(g["seed"]))
    np.testing.assert_allclose(checksum(system), g["checksum"], rtol=1e-13)
    cfg = SolverConfig(p=int(g["p"]), depth=int(g["depth"]), precision=precision)
    st = Stepper(system, lam.values, cfg)
    for _ in range(2):
        e, f, lf = st.step(system.positions)
    tol = TOL[precision]
    idx = g["idx"]
    sidx, dforce, _ = site_force_fixture("c3" if case == "c3d6" else case)
    f_ref = g["forces"].copy()
    pos_in_sample = {int(a): k for k, a in enumerate(idx)}
    hit = 0
    for a, df in zip(sidx, dforce):
        k = pos_in_sample.get(int(a))
        if k is not None:
            f_ref[k] += df
            hit += 1
    err = {
        "energy": abs(e - float(g["hi_energy"])) / abs(float(g["hi_energy"])),
        "lambda_forces": relerr(lambda_rows(system, lam.values, lf), g["hi_forces"]),
        "forces": float(np.max(np.abs(f[idx] - f_ref)) / g["absmax_forces"]),
    }
    # every site atom: the reference's spatial force is not in the fixture
    # for atoms outside the sample, so check the site term by difference
    # with the device's own charge-scaled forces
    qi = hi_energy_and_forces(system, lam.values, solver=st.solver, mode="qi", spatial_forces=True)
    err["site_term"] = relerr(f[sidx] - qi.spatial_forces[sidx], dforce)
    print(case, precision, "sample site atoms", hit, {k: "%.2e" % v for k, v in err.items()})
    assert err["energy"] <= tol and err["lambda_forces"] <= tol and err["forces"] <= tol
    assert err["site_term"] <= 1e-6


@pytest.mark.slow
def test_step_tree_c3_bit_exact():
    """The tree the benchmarked step rebuilds at C3 (1M atoms, depth 5) and
    the depth-6 tree of the same box: perm and leaf_start bit-identical to
    the reference's build_octree (sha256)."""
    g = np.load(os.path.join(GOLDEN, "ref_trees.npz"))
    system, lam = water(1_000_000, 512, 4)
    np.testing.assert_allclose(checksum(system), g["c3_checksum"], rtol=1e-13)
    for d in (5, 6):
        st = Stepper(system, lam.values, SolverConfig(p=10, depth=d, precision="single"))
        st.step(system.positions)
        hp, hl, perm = st.tree_hashes()
        np.testing.assert_array_equal(perm[:4096], g[f"c3_d{d}_perm_head"])
        assert hp == str(g[f"c3_d{d}_perm_sha"]) and hl == str(g[f"c3_d{d}_leaf_start_sha"]), d


# -------------------------------------------- tree rebuilt across MD steps ----
def moved_positions(system, step, sigma=0.01, seed=77):
    """tests/golden/make_golden_large.py moved_positions, same sequence."""
    rng = np.random.default_rng(seed)
    pos = np.array(system.positions, dtype=np.float64)
    for _ in range(step):
        pos = pos + rng.normal(0.0, sigma, pos.shape)
    return pos


@pytest.mark.slow
def test_tree_rebuilt_across_steps_c2_bit_exact():
    """one plan, positions moving every step (unwrapped
    random walk, sigma 0.01 nm); after each lfmm_step the exported tree is the
    reference's build_octree of that step's positions, bit for bit."""
    g = np.load(os.path.join(GOLDEN, "ref_trees.npz"))
    system, lam = water(100_000, 64, 3)
    np.testing.assert_allclose(checksum(system), g["c2_checksum"], rtol=1e-13)
    for precision in ("single", "double"):
        st = Stepper(system, lam.values, SolverConfig(p=10, depth=4, precision=precision))
        for k in (0, 1, 2, 3, 1):
            st.step(moved_positions(system, k))
            hp, hl, perm = st.tree_hashes()
            np.testing.assert_array_equal(perm[:4096], g[f"c2_step{k}_perm_head"])
            assert hp == str(g[f"c2_step{k}_perm_sha"]), (precision, k)
            assert hl == str(g[f"c2_step{k}_leaf_start_sha"]), (precision, k)


@pytest.mark.parametrize("precision", ["double", "single"])
def test_step_values_follow_moving_atoms(precision):
    """C1 box over three MD-like steps on one plan: each step's energy,
    forces and lambda forces equal the oracle at that step's positions (the
    oracle builds a fresh tree each time, like a fresh PeriodicSolver)."""
    system, lam = water(3000, 4, 0)
    cfg = SolverConfig(p=8, depth=3, precision=precision)
    ocfg = orc.default_config(p=8, depth=3)
    sites = [(s.particle_indices, s.form_charges) for s in system.sites]
    st = Stepper(system, lam.values, cfg)
    tol = TOL[precision]
    for k in (1, 2, 3):
        pos = moved_positions(system, k, sigma=0.03)
        ref = orc.hi(pos, system.charges, system.box_length, sites, lam.values, ocfg)
        fq = orc.solve(pos, ref["q_tilde"], system.box_length, ocfg, forces=True)["forces"]
        # the HI correction reads the caller's (unwrapped) site positions,
        # as corrections.py:173 does
        fq[np.concatenate([s[0] for s in sites])] += orc.hi_site_forces(
            pos, system.box_length, sites, lam.values, ocfg, ref["solve"]["lattice"])
        e, f, lf = st.step(pos)
        assert relerr(e, ref["energy"]) <= tol, k
        assert relerr(f, fq) <= tol, k
        assert relerr(lambda_rows(system, lam.values, lf), np.concatenate(ref["forces"])) <= tol, k


# ------------------------------------------------- HI spatial forces, FD ----
def small_sites_system(seed=11, n_bg=300, box=3.2, nsites=3, ns=6):
    from paper_2410_01754_b200.system import LambdaState, ParticleSystem, TitratableSite

    rng = np.random.default_rng(seed)
    pos = [rng.uniform(0, box, (n_bg, 3))]
    q = [rng.uniform(-0.5, 0.5, n_bg)]
    sites = []
    for s in range(nsites):
        c = rng.uniform(0.6, box - 0.6, 3)
        pos.append(c + rng.uniform(-0.25, 0.25, (ns, 3)))
        q.append(np.zeros(ns))
        nf = 2 if s % 2 == 0 else 4
        sites.append(TitratableSite(np.arange(n_bg + s * ns, n_bg + (s + 1) * ns), rng.uniform(-0.6, 0.6, (nf, ns))))
    system = ParticleSystem(box, np.vstack(pos), np.concatenate(q), sites)
    lam = LambdaState(values=[rng.uniform(0.15, 0.85, int(np.log2(s.num_forms))) for s in sites],
                      velocities=[np.zeros(int(np.log2(s.num_forms))) for s in sites], masses=[5.0] * nsites)
    return system, lam


@pytest.mark.parametrize("kw", [dict(), dict(intra_site_images="minimum"),
                                dict(lattice_mode="shells", shell_cap=3, dipole=False),
                                dict(lattice_mode="off", dipole=True), dict(depth=1)])
def test_hi_spatial_forces_match_finite_difference(kw):
    """-dE_HI/dr by central differences of hi_energy_and_forces(...).energy
    (h = 1e-6, atol 5e-7: the reference's own spatial-force FD protocol,
    test_fmm_engine.py:113-128) on every site atom and a few environment
    atoms, against the analytic forces of the same call (fp64)."""
    system, lam = small_sites_system()
    kw = dict(kw)
    cfg = SolverConfig(p=14, depth=kw.pop("depth", 0), **kw)
    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    r = hi_energy_and_forces(system, lam.values, solver=solver, spatial_forces=True)
    atoms = list(np.concatenate([s.particle_indices for s in system.sites])) + [0, 7, 150]
    h = 1e-6
    worst = 0.0
    for a in atoms:
        for x in range(3):
            e = []
            for sgn in (1, -1):
                s2 = copy.copy(system)
                s2.positions = np.array(system.positions)
                s2.positions[a, x] += sgn * h
                sv = PeriodicSolver(s2.positions, s2.box_length, cfg)
                e.append(hi_energy_and_forces(s2, lam.values, solver=sv).energy)
            fd = -(e[0] - e[1]) / (2 * h)
            worst = max(worst, abs(fd - r.spatial_forces[a, x]))
    assert worst <= 5e-7, worst


def test_hi_site_forces_match_reference_fixture():
    """The device site term alone (lfmm_hi_site_forces) against the
    reference's central differences at C1, full and minimum images."""
    system, lam = water(3000, 4, 0)
    for images, tag in (("full", "c1"), ("minimum", "c1_minimum")):
        idx, dforce, ck = site_force_fixture(tag)
        np.testing.assert_allclose(ck, checksum(system), rtol=1e-13)
        solver = PeriodicSolver(system.positions, system.box_length,
                                SolverConfig(p=8, depth=3, intra_site_images=images))
        r = hi_energy_and_forces(system, lam.values, solver=solver, spatial_forces=True)
        assert relerr(solver.plan.hi_site_forces(), dforce) <= 1e-9
        np.testing.assert_array_equal(idx, np.concatenate([s.particle_indices for s in system.sites]))
        assert r.spatial_forces is not None


def test_overlapping_sites_rejected():
    """Sites may not share particles (system.py:135-143); the site-force add
    relies on it."""
    from paper_2410_01754_b200.system import ParticleSystem, TitratableSite

    system, lam = small_sites_system()
    s0 = system.sites[0]
    bad = ParticleSystem(system.box_length, system.positions, system.charges,
                         [s0, TitratableSite(np.array(s0.particle_indices), s0.form_charges)])
    solver = PeriodicSolver(bad.positions, bad.box_length, SolverConfig(p=6, depth=1))
    with pytest.raises(ValueError, match="overlap"):
        hi_energy_and_forces(bad, [lam.values[0], lam.values[0]], solver=solver)


def test_host_input_step_matches_device_input_step():
    """lfmm_step with host buffers (bench.py's e2e call: positions uploaded in
    four pieces, each counted as it lands; charges on the io stream; forces
    downloaded beside the HI tail) gives the device-input step's results bit
    for bit, on a system large enough (>= 2^18 atoms) for the chunked upload,
    and rebuilds the same tree."""
    system, lam, _ = generate_water_box(300_000, 32, seed=5)
    cfg = SolverConfig(p=10, depth=4, precision="single")
    st = Stepper(system, lam.values, cfg)
    e_dev, f_dev, lf_dev = st.step(system.positions)
    h_dev = st.tree_hashes()[:2]
    lt, nl = lambda_table(system, lam.values)
    n, s = system.num_particles, len(system.sites)
    e = np.empty(1)
    f = np.empty((n, 3))
    lf = np.empty((s, 4))
    for _ in range(2):  # the second call reuses the plan's io stream and events
        st.plan.step(np.ascontiguousarray(system.positions), np.ascontiguousarray(system.charges), lt, nl,
                     mode=_native.MODE_HI, plain=False, on_device=False, energy=e, forces=f, lambda_forces=lf)
        assert st.tree_hashes()[:2] == h_dev
        assert e[0] == e_dev
        np.testing.assert_array_equal(f, f_dev)
        np.testing.assert_array_equal(lf, lf_dev)
