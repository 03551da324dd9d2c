"""Golden fixtures at the benchmark sizes (C2, C3), made by the REFERENCE.

SURVEY.md §8c step 4: at C3 compare energies, lambda-forces and a 10k-atom
sample of potentials/forces against the reference itself.  The water boxes
are regenerated bit-identically from their seeds on the GPU box
(paper_2410_01754_b200/waterbox.py, numpy default_rng), so the fixture stores
only a checksum of the inputs plus the reference's outputs on a sample.

Run in the build container (where /root/reference exists; ~6 min on 8 cores):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden_large.py
"""

import hashlib
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

from lambdafmm import corrections as rc  # noqa: E402
from lambdafmm.fmm.octree import build_octree  # noqa: E402
from lambdafmm.system import wrap_positions  # noqa: E402
from lambdafmm.fmm.solver import PeriodicSolver, SolverConfig  # noqa: E402
from lambdafmm.system import scale_charges as rscale  # noqa: E402
from lambdafmm.weights import expand_weights as rexp  # noqa: E402

from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
NSAMPLE = 10_000


def checksum(system):
    return np.array([system.positions.sum(), (system.positions ** 2).sum(), system.charges.sum(),
                     np.abs(system.charges).sum(), float(system.num_particles)])


def make(name, n_atoms, n_sites, seed, depth):
    t0 = time.time()
    system, lam, _ = generate_water_box(n_atoms, n_sites, seed=seed)
    cfg = SolverConfig(p=10, depth=depth)
    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    r = rc.hi_energy_and_forces(system, lam.values, solver=solver)
    qt = rscale(system, [rexp(v) for v in lam.values])
    forces = solver.spatial_forces(qt)
    n = system.num_particles
    idx = np.sort(np.random.default_rng(1234).choice(n, size=min(NSAMPLE, n), replace=False))
    s = r.solve
    arrs = dict(
        n_atoms=n_atoms, n_sites=n_sites, seed=seed, p=cfg.p, depth=depth, checksum=checksum(system), idx=idx,
        potentials=s.potentials[idx], near=s.near_potentials[idx], far=s.far_potentials[idx],
        dip=s.dipole_potentials[idx], forces=forces[idx],
        absmax_potentials=np.abs(s.potentials).max(), absmax_near=np.abs(s.near_potentials).max(),
        absmax_far=np.abs(s.far_potentials).max(), absmax_dip=np.abs(s.dipole_potentials).max(),
        absmax_forces=np.abs(forces).max(),
        energy=s.energy, near_energy=s.near_energy, far_energy=s.far_energy, dipole_energy=s.dipole_energy,
        hi_energy=r.energy, hi_forces=np.concatenate(r.forces),
        c_p2p=np.concatenate([c.c_p2p for c in r.corrections.sites]),
        c_lattice=np.concatenate([c.c_lattice for c in r.corrections.sites]),
        c_dipole=np.concatenate([c.c_dipole for c in r.corrections.sites]),
        reference_seconds=time.time() - t0, cpu_count=os.cpu_count())
    np.savez_compressed(os.path.join(OUT, name), **arrs)
    print("wrote", name, "in %.1f s" % (time.time() - t0))


def tree_hashes(positions, box_length, depth):
    """sha256 of the reference's canonical permutation and leaf CSR
    (octree.build_octree, octree.py:114-163) for a bit-exact check."""
    t = build_octree(wrap_positions(positions, box_length), box_length, depth)
    return (hashlib.sha256(np.ascontiguousarray(t.perm, dtype=np.int64).tobytes()).hexdigest(),
            hashlib.sha256(np.ascontiguousarray(t.leaf_start, dtype=np.int64).tobytes()).hexdigest(),
            np.asarray(t.perm[:4096], dtype=np.int64))


def moved_positions(system, step, sigma=0.01, seed=77):
    """Positions after `step` deterministic random displacements (an MD-like
    trajectory for the per-step tree rebuild); unwrapped
    on purpose: the solver wraps them (system.py:103-108)."""
    rng = np.random.default_rng(seed)
    pos = np.array(system.positions, dtype=np.float64)
    for _ in range(step):
        pos = pos + rng.normal(0.0, sigma, pos.shape)
    return pos


def site_delta_energy(pos, qf, lams, box_length, lattice_matrix, p, images, dipole):
    """Delta E_site = e(q~) - sum_rho w_rho C_rho of one site, from the
    reference's own per-site pieces (corrections.py:157-193)."""
    w = rexp(lams)
    cc = rc.correction_charges(qf, w)
    kern = rc.near_kernel(pos, box_length, images)
    c = np.einsum("fs,st,ft->f", qf, kern, cc.half_offset)
    eb = 0.5 * float(cc.blend @ kern @ cc.blend)
    if images == "full" and lattice_matrix is not None:
        g = rc.lattice_kernel(pos, box_length, lattice_matrix, p)
        c = c + np.einsum("fs,st,ft->f", qf, g, cc.half_offset)
        eb += 0.5 * float(cc.blend @ g @ cc.blend)
    if images == "full" and dipole:
        c = c + rc.c_dipole(pos, qf, w, box_length)
    return eb - float(w.values @ c)


def site_force_corrections(system, lam_values, solver, sites, h=1e-4):
    """-dDelta E_site/dr of every atom of the chosen sites by the 4-point
    central difference (O(h^4)); the HI spatial forces on site atoms are
    spatial_forces(q~) plus these."""
    cfg = solver.config
    out_idx, out_f = [], []
    for s in sites:
        site = system.sites[s]
        pos0 = np.array(system.positions[site.particle_indices], dtype=np.float64)
        args = (site.form_charges, lam_values[s], system.box_length, solver.lattice_matrix, cfg.p,
                cfg.intra_site_images, cfg.dipole)
        f = np.zeros_like(pos0)
        for a in range(pos0.shape[0]):
            for x in range(3):
                e = []
                for k in (-2, -1, 1, 2):
                    pp = pos0.copy()
                    pp[a, x] += k * h
                    e.append(site_delta_energy(pp, *args))
                f[a, x] = -(e[0] - 8 * e[1] + 8 * e[2] - e[3]) / (12 * h)
        out_idx.append(site.particle_indices)
        out_f.append(f)
    return np.concatenate(out_idx), np.concatenate(out_f)


def make_trees():
    """Reference tree hashes: the C3 box at depth 5 and 6, and the C2 box
    moved over three MD-like steps at depth 4 (per-step rebuild)."""
    arrs = {}
    system, _, _ = generate_water_box(1_000_000, 512, seed=4)
    arrs["c3_checksum"] = checksum(system)
    for d in (5, 6):
        hp, hl, head = tree_hashes(system.positions, system.box_length, d)
        arrs[f"c3_d{d}_perm_sha"], arrs[f"c3_d{d}_leaf_start_sha"], arrs[f"c3_d{d}_perm_head"] = hp, hl, head
    system, _, _ = generate_water_box(100_000, 64, seed=3)
    arrs["c2_checksum"] = checksum(system)
    for k in range(4):
        pos = moved_positions(system, k)
        hp, hl, head = tree_hashes(pos, system.box_length, 4)
        arrs[f"c2_step{k}_perm_sha"], arrs[f"c2_step{k}_leaf_start_sha"], arrs[f"c2_step{k}_perm_head"] = hp, hl, head
    np.savez_compressed(os.path.join(OUT, "ref_trees.npz"), **arrs)
    print("wrote ref_trees.npz")


def make_site_forces():
    """Reference -dDelta E_site/dr at C1 (all sites, fp64 configs of the
    fixtures), C2 (all 64 sites) and C3 (all 512 sites)."""
    arrs = {}
    for tag, (n, ns, seed, p, d) in {"c1": (3000, 4, 0, 8, 3), "c2": (100_000, 64, 3, 10, 4),
                                     "c3": (1_000_000, 512, 4, 10, 5)}.items():
        t0 = time.time()
        system, lam, _ = generate_water_box(n, ns, seed=seed)
        for images in ("full", "minimum"):
            if images == "minimum" and tag != "c1":
                continue
            cfg = SolverConfig(p=p, depth=d, intra_site_images=images)
            # the lattice operator only: a 1-atom solver carries the same matrix
            solver = PeriodicSolver(system.positions[:1], system.box_length, cfg)
            idx, f = site_force_corrections(system, lam.values, solver, range(len(system.sites)))
            key = tag if images == "full" else tag + "_minimum"
            arrs[key + "_checksum"] = checksum(system)
            arrs[key + "_idx"] = idx
            arrs[key + "_dforce"] = f
        print(tag, "site forces in %.1f s" % (time.time() - t0))
    np.savez_compressed(os.path.join(OUT, "ref_site_forces.npz"), **arrs)
    print("wrote ref_site_forces.npz")


def make_site_forces_c4():
    """The C4 box (4096 sites): -dDelta E_site/dr of every site atom."""
    t0 = time.time()
    system, lam, _ = generate_water_box(1_000_000, 4096, seed=5)
    solver = PeriodicSolver(system.positions[:1], system.box_length, SolverConfig(p=10, depth=5))
    idx, f = site_force_corrections(system, lam.values, solver, range(len(system.sites)))
    np.savez_compressed(os.path.join(OUT, "ref_site_forces_c4.npz"), c4_checksum=checksum(system), c4_idx=idx,
                        c4_dforce=f)
    print("c4 site forces in %.1f s" % (time.time() - t0))


def main():
    which = sys.argv[1:] or ["c2", "c3"]
    if "c2" in which:
        make("ref_c2_d4.npz", 100_000, 64, 3, 4)
    if "c3" in which:
        make("ref_c3_d5.npz", 1_000_000, 512, 4, 5)
    if "trees" in which:
        make_trees()
    if "sitef" in which:
        make_site_forces()
    if "c4" in which:
        # the HI site-count stress box
        make("ref_c4_d5.npz", 1_000_000, 4096, 5, 5)
    if "sitef4" in which:
        make_site_forces_c4()
    if "c3d6" in which:
        # the C3 box at the reference's depth cap (solver.py:62-64), ~3.8 atoms/leaf
        make("ref_c3_d6.npz", 1_000_000, 512, 4, 6)


if __name__ == "__main__":
    main()
