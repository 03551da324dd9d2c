"""Golden fixtures at the benchmark sizes (C2, C3), made by the REFERENCE.

SURVEY.md §8c step 4: at C3 compare energies, lambda-forces and a 10k-atom
sample of potentials/forces against the reference itself.  The water boxes
are regenerated bit-identically from their seeds on the GPU box
(paper_2410_01754_b200/waterbox.py, numpy default_rng), so the fixture stores
only a checksum of the inputs plus the reference's outputs on a sample.

Run in the build container (where /root/reference exists; ~6 min on 8 cores):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden_large.py
"""

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


def main():
    which = sys.argv[1:] or ["c2", "c3"]
    if "c2" in which:
        make("ref_c2_d4.npz", 100_000, 64, 3, 4)
    if "c3" in which:
        make("ref_c3_d5.npz", 1_000_000, 512, 4, 5)


if __name__ == "__main__":
    main()
