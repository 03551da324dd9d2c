"""Relative errors (max-normalised) of the fp32 path vs the reference golden
fixtures, for the M2L kernel selected by LFMM_M2L (default: tensor cores)."""
import glob
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "tests")))
from conftest import load_golden, relerr  # noqa: E402
from test_gpu_hi import cfg_from as hcfg, system_from  # noqa: E402
from test_gpu_solve import cfg_from as scfg  # noqa: E402

from paper_2410_01754_b200 import PeriodicSolver, hi_energy_and_forces  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "single"
for path in sorted(glob.glob("tests/golden/solve_*.npz")):
    g = load_golden(os.path.basename(path))
    s = PeriodicSolver(g["positions"], float(g["box"]), scfg(g, prec))
    r = s.solve(g["charges"])
    print(f"{os.path.basename(path):28s} pot {relerr(r.potentials, g['potentials']):.2e} far {relerr(r.far_potentials, g['far']):.2e} "
          f"E {relerr(r.energy, g['energy']):.2e} Efar {relerr(r.far_energy, g['far_energy']):.2e}")
for path in sorted(glob.glob("tests/golden/hi_*.npz")):
    g = load_golden(os.path.basename(path))
    system, lam = system_from(g)
    solver = PeriodicSolver(system.positions, system.box_length, hcfg(g, prec))
    r = hi_energy_and_forces(system, lam, solver=solver)
    rq = hi_energy_and_forces(system, lam, solver=solver, mode="qi")
    print(f"{os.path.basename(path):28s} E_hi {relerr(r.energy, g['hi_energy']):.2e} F_hi {relerr(np.concatenate(r.forces), g['hi_forces']):.2e} "
          f"E_qi {relerr(rq.energy, g['qi_energy']):.2e} pot {relerr(r.solve.potentials, g['potentials']):.2e}")
