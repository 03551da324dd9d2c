"""Diagnostic (not a test): fp32 vs fp64 errors at C3 for each M2L path and
lattice mode; predicted constant offset from the lattice root local."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig
from paper_2410_01754_b200.waterbox import generate_water_box

def relerr(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 5
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["halo", "gather"]
system, lam, _ = generate_water_box(n, 8, seed=4)
for lat in ("converged", "off"):
    s64 = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=depth, lattice_mode=lat))
    r64 = s64.solve(system.charges)
    print("lattice", lat, "max|pot| %.4g max|far| %.4g" % (np.max(np.abs(r64.potentials)), np.max(np.abs(r64.far_potentials))))
    for mode in modes:
        os.environ["LFMM_M2L"] = mode
        s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=depth, lattice_mode=lat, precision="single"))
        r = s.solve(system.charges)
        print(" ", mode, {k: "%.3e" % relerr(getattr(r, k), getattr(r64, k)) for k in ("potentials", "far_potentials", "near_potentials", "energy", "far_energy", "root_multipole")})
        d = r.far_potentials - r64.far_potentials
        msg = "   far err mean %.3e std %.3e" % (d.mean(), d.std())
        if s64.lattice_matrix is not None:
            dm = r.root_multipole - r64.root_multipole
            pred = np.real(s64.lattice_matrix[0] @ dm)
            msg += "  predicted lattice offset %.3e" % pred
            nc = dm.size
            ls = np.floor(np.sqrt(np.arange(nc))).astype(int)
            for l in range(0, 11, 2):
                sel = ls == l
                msg += "\n     l=%d |dM|max %.3e |M|max %.3e" % (l, np.abs(dm[sel]).max(), np.abs(r64.root_multipole[sel]).max())
        print(msg)
os.environ.pop("LFMM_M2L", None)
