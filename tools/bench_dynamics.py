"""Device-resident lambda dynamics at C3 (1M atoms, 512 sites, p=10, d=5,
fp32): ms per BAOAB step of run_trajectory_device (engine step with the tree
frozen + the two k_lambda_baoab kicks), against the same step driven from
the host with EngineLambdaForceField (lambdas and forces round-trip)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_01754_b200 import dynamics as dyn  # noqa: E402
from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig  # noqa: E402
from paper_2410_01754_b200.system import LambdaState  # noqa: E402
from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

system, lam, _ = generate_water_box(1_000_000, 512, seed=0)
state = LambdaState(values=[np.asarray(v, float) for v in lam.values],
                    velocities=[np.zeros(len(v)) for v in lam.values], masses=[5.0] * len(lam.values))
solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=5, precision="single"))
dyn.run_trajectory_device(system, state.copy(), 5, solver=solver, sample_every=5)
torch.cuda.synchronize()
n = 50
t0 = time.perf_counter()
dyn.run_trajectory_device(system, state.copy(), n, solver=solver, sample_every=10)
torch.cuda.synchronize()
dev_ms = (time.perf_counter() - t0) * 1e3 / n
field = dyn.EngineLambdaForceField(system, solver=solver)
dyn.run_trajectory(field, state.copy(), 2)
t0 = time.perf_counter()
dyn.run_trajectory(field, state.copy(), 10, sample_every=10)
host_ms = (time.perf_counter() - t0) * 1e3 / 10
print(f"device BAOAB loop: {dev_ms:.3f} ms/step (wall, incl. launch overhead); host loop with "
      f"EngineLambdaForceField: {host_ms:.3f} ms/step")
