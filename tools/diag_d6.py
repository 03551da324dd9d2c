"""Depth-6 diagnosis: one fp32 (or fp64) solve on a 300k-atom box, timed."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig  # noqa: E402
from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "single"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300_000
system, _, _ = generate_water_box(n, 0, seed=6)
t = time.time()
s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=6, precision=prec))
print(prec, "plan", round(time.time() - t, 2), "s", flush=True)
t = time.time()
r = s.solve(system.charges)
print(prec, "solve", round(time.time() - t, 2), "s energy", float(r.energy), flush=True)
np.save(f"gpurun_out/d6_{prec}.npy", r.potentials)
