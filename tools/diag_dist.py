import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from test_gpu_distributed import _single, _distributed
from paper_2410_01754_b200.fmm.solver import SolverConfig, PeriodicSolver
from paper_2410_01754_b200.waterbox import generate_water_box
system, lam, _ = generate_water_box(40_000, 24, seed=11)
cfg = SolverConfig(p=10, depth=4, precision=sys.argv[1] if len(sys.argv) > 1 else "double")
e1, f1, lf1 = _single(system, lam.values, cfg)
s = PeriodicSolver(system.positions, system.box_length, cfg)
from paper_2410_01754_b200 import hi_energy_and_forces
r = hi_energy_and_forces(system, lam.values, solver=s)
print("single step energy", e1, " hi_energy_and_forces", r.energy, "solve", r.solve.energy, r.solve.near_energy, r.solve.far_energy, r.solve.dipole_energy)
for world in (1, 2):
    outs, fd = _distributed(system, lam.values, cfg, world) if world > 1 else (None, None)
    if outs is None: continue
    for o in outs:
        print(world, {k: (round(v, 10) if isinstance(v, float) else None) for k, v in o.items() if isinstance(v, float)})
    print("force relerr", np.max(np.abs(fd - f1)) / np.max(np.abs(f1)))
    for o in outs: print("lf relerr", np.max(np.abs(o["lambda_forces"].cpu().numpy() - lf1)) / np.max(np.abs(lf1)))
