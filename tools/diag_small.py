"""Diagnostic: fp32 vs fp64 energy pieces on a golden fixture, per P2P kernel."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig
name = sys.argv[1] if len(sys.argv) > 1 else "hi_small_minimum.npz"
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", name))
cfg = dict(p=int(g["p"]), depth=int(g["depth"]), lattice_mode=str(g["lattice_mode"]), shell_cap=int(g["shell_cap"]), dipole=bool(g["dipole"]))
r64 = PeriodicSolver(g["positions"], float(g["box"]), SolverConfig(**cfg)).solve(g["charges"])
for kern in ("packed", "scalar"):
    os.environ["LFMM_P2P"] = kern
    r = PeriodicSolver(g["positions"], float(g["box"]), SolverConfig(precision="single", **cfg)).solve(g["charges"])
    print(kern, "E rel %.2e | near %.2e far %.2e dip %.2e (abs) | Vnear maxabs err %.2e" % (
        abs(r.energy - r64.energy) / abs(r64.energy), r.near_energy - r64.near_energy, r.far_energy - r64.far_energy,
        r.dipole_energy - r64.dipole_energy, np.abs(r.near_potentials - r64.near_potentials).max()))
