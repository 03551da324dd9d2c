"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

Every fixture stores its inputs and the reference's outputs; the tests
never import the reference (it does not exist on the GPU box).
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

from lambdafmm import corrections as rc  # noqa: E402
from lambdafmm.fmm import octree as ro  # noqa: E402
from lambdafmm.fmm.solver import PeriodicSolver, SolverConfig  # noqa: E402
from lambdafmm.system import ParticleSystem, TitratableSite  # noqa: E402

from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrs):
    np.savez_compressed(os.path.join(OUT, name), **arrs)
    print("wrote", name, sum(np.asarray(a).nbytes for a in arrs.values()), "bytes raw")


def cloud(n, box, seed):
    g = np.random.default_rng(seed)
    pos = g.uniform(0, box, size=(n, 3))
    q = g.uniform(-1, 1, size=n)
    q -= q.mean()
    return pos, q


def tree_fixture(name, n, box, depth, seed):
    pos, _ = cloud(n, box, seed)
    # add exact duplicates / ties in x to exercise the lexsort tie-breaks
    pos[5] = pos[3]
    pos[7, 0] = pos[8, 0]
    t = ro.build_octree(pos, box, depth)
    arrs = dict(positions=pos, box=box, depth=depth, perm=t.perm, inv_perm=t.inv_perm, leaf_start=t.leaf_start,
                leaf_of_particle=t.leaf_of_particle, positions_sorted=t.positions, nb_box=t.nb_box,
                nb_shift=t.nb_shift)
    for l in range(1, depth + 1):
        rows, cnt, tg, sr = [], [], [], []
        for row, targets, sources in t.levels[l].m2l:
            rows.append(row)
            cnt.append(targets.size)
            tg.append(targets)
            sr.append(sources)
        arrs[f"m2l{l}_rows"] = np.array(rows)
        arrs[f"m2l{l}_counts"] = np.array(cnt)
        arrs[f"m2l{l}_targets"] = np.concatenate(tg)
        arrs[f"m2l{l}_sources"] = np.concatenate(sr)
    for l in range(depth):
        arrs[f"child{l}"] = t.levels[l].child_index
    save(name, **arrs)


def solve_fixture(name, pos, q, box, cfg, forces=True):
    s = PeriodicSolver(pos, box, cfg)
    r = s.solve(q)
    arrs = dict(positions=pos, charges=q, box=box, p=cfg.p, depth=cfg.depth, lattice_mode=cfg.lattice_mode,
                shell_cap=cfg.shell_cap, dipole=cfg.dipole, periodic_near=cfg.periodic_near,
                potentials=r.potentials, near=r.near_potentials, far=r.far_potentials, dip=r.dipole_potentials,
                energy=r.energy, near_energy=r.near_energy, far_energy=r.far_energy,
                dipole_energy=r.dipole_energy, root_multipole=r.root_multipole, dipole_vector=r.dipole_vector,
                total_charge=r.total_charge)
    if s.lattice_matrix is not None:
        arrs["lattice_matrix"] = s.lattice_matrix
    if forces and np.ndim(q) == 1:
        arrs["forces"] = s.spatial_forces(q)
    save(name, **arrs)


def hi_fixture(name, system, lam_values, cfg):
    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    r = rc.hi_energy_and_forces(system, lam_values, solver=solver)
    rq = rc.hi_energy_and_forces(system, lam_values, solver=solver, mode="qi")
    sites = system.sites
    arrs = dict(positions=system.positions, charges=system.charges, box=system.box_length, p=cfg.p,
                depth=cfg.depth, lattice_mode=cfg.lattice_mode, shell_cap=cfg.shell_cap, dipole=cfg.dipole,
                intra=cfg.intra_site_images,
                site_atom_offsets=np.concatenate([[0], np.cumsum([s.num_particles for s in sites])]),
                site_atoms=np.concatenate([s.particle_indices for s in sites]),
                site_nforms=np.array([s.num_forms for s in sites]),
                site_forms=np.concatenate([s.form_charges.reshape(-1) for s in sites]),
                lambdas=np.concatenate([np.asarray(v, float) for v in lam_values]),
                n_lambda=np.array([len(v) for v in lam_values]),
                hi_energy=r.energy, qi_energy=rq.energy,
                hi_forces=np.concatenate(r.forces), qi_forces=np.concatenate(rq.forces),
                c_p2p=np.concatenate([c.c_p2p for c in r.corrections.sites]),
                c_lattice=np.concatenate([c.c_lattice for c in r.corrections.sites]),
                c_dipole=np.concatenate([c.c_dipole for c in r.corrections.sites]),
                blend=np.array([c.blend_energy for c in r.corrections.sites]),
                offset=r.corrections.energy_offset(), potentials=r.solve.potentials,
                solve_energy=r.solve.energy)
    save(name, **arrs)


def small_hi_system(seed=77, box=4.0, nforms=(2, 4), ns=4, n_bg=60):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0, box, (n_bg, 3))
    q = rng.uniform(-0.5, 0.5, n_bg)
    q -= q.mean()
    sites, allp = [], [pos]
    for s, nf in enumerate(nforms):
        c = rng.uniform(0, box, 3)
        sp = (c + rng.uniform(-0.25, 0.25, (ns, 3))) % box
        allp.append(sp)
        sites.append(TitratableSite(np.arange(n_bg + s * ns, n_bg + (s + 1) * ns), rng.uniform(-0.5, 0.5, (nf, ns))))
    return ParticleSystem(box, np.vstack(allp), np.concatenate([q, np.zeros(len(nforms) * ns)]), sites)


def main():
    tree_fixture("tree_d3.npz", 400, 2.0, 3, seed=1)
    tree_fixture("tree_d1.npz", 50, 1.0, 1, seed=2)
    pos, q = cloud(40, 2.0, 1)
    solve_fixture("solve_d0_off.npz", pos, q, 2.0, SolverConfig(p=6, depth=0, lattice_mode="off", dipole=False))
    pos, q = cloud(64, 3.0, 7)
    solve_fixture("solve_d2_conv_p9.npz", pos, q, 3.0, SolverConfig(p=9, depth=2))
    pos, q = cloud(60, 3.0, 2)
    solve_fixture("solve_d1_shells_p16.npz", pos, q, 3.0,
                  SolverConfig(p=16, depth=1, lattice_mode="shells", shell_cap=3, dipole=False))
    pos, q = cloud(20, 2.0, 10)
    solve_fixture("solve_d0_conv_p14.npz", pos, q, 2.0, SolverConfig(p=14, depth=0))
    g = np.random.default_rng(6)
    pos, _ = cloud(35, 2.0, 5)
    solve_fixture("solve_multi_rhs.npz", pos, g.uniform(-1, 1, size=(35, 4)), 2.0, SolverConfig(p=10, depth=1),
                  forces=False)
    # C1: ~3k-atom water box, 4 sites, p=8, depth 3
    system, lam, info = generate_water_box(3000, 4, seed=0)
    cfg = SolverConfig(p=8, depth=3)
    from lambdafmm.system import scale_charges as rscale
    from lambdafmm.weights import expand_weights as rexp
    qt = rscale(system, [rexp(v) for v in lam.values])
    solve_fixture("solve_c1_water.npz", system.positions, qt, system.box_length, cfg)
    hi_fixture("hi_c1_water.npz", system, lam.values, cfg)
    hs = small_hi_system()
    hi_fixture("hi_small_conv.npz", hs, [[0.345], [0.3, 0.8]], SolverConfig(p=8, depth=1))
    hi_fixture("hi_small_minimum.npz", hs, [[0.345], [0.3, 0.8]],
               SolverConfig(p=8, depth=0, intra_site_images="minimum"))
    hi_fixture("hi_small_nodip_shells.npz", hs, [[0.7], [0.25, 0.6]],
               SolverConfig(p=10, depth=1, lattice_mode="shells", shell_cap=3, dipole=False))


if __name__ == "__main__":
    main()
