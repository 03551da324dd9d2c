"""Host-side cost of one lfmm_step call (device-resident inputs) vs its GPU time:
if the host needs longer to enqueue a step than the GPU to run it, the GPU idles."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_01754_b200 import _native  # noqa: E402
from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig  # noqa: E402
from paper_2410_01754_b200.system import lambda_table, site_tables  # noqa: E402
from paper_2410_01754_b200.waterbox import generate_water_box  # noqa: E402

system, lam_state, _ = generate_water_box(1_000_000, 512, seed=0)
dev = torch.device("cuda", 0)
solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=5, precision="single"))
plan = solver.plan
plan.set_sites(*site_tables(system))
lam, nl = lambda_table(system, lam_state.values)
stream = torch.cuda.Stream(device=dev)
plan.set_stream(stream.cuda_stream)
n, s = system.num_particles, len(system.sites)
d_pos = torch.from_numpy(np.ascontiguousarray(system.positions)).to(dev)
d_q = torch.from_numpy(np.ascontiguousarray(system.charges)).to(dev)
d_lam = torch.from_numpy(lam).to(dev)
d_nl = torch.from_numpy(nl).to(dev)
d_e = torch.empty(1, dtype=torch.float64, device=dev)
d_f = torch.empty((n, 3), dtype=torch.float64, device=dev)
d_lf = torch.empty((s, 4), dtype=torch.float64, device=dev)


def step():
    plan.step(d_pos, d_q, d_lam, d_nl, mode=_native.MODE_HI, plain=False, on_device=True, energy=d_e, forces=d_f,
              lambda_forces=d_lf)


for _ in range(5):
    step()
torch.cuda.synchronize()
K = 50
t0 = time.perf_counter()
for _ in range(K):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3 * (t1 - t0) / K:.3f} ms/step, wall incl. GPU {1e3 * (t2 - t0) / K:.3f} ms/step")
