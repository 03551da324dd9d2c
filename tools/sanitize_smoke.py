"""Small C1-sized workload for compute-sanitizer: solve + forces + HI step in
fp64 and fp32 (tcgen05 M2L, preemptible P2P at depth 3), bench-style step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig, hi_energy_and_forces, _native
from paper_2410_01754_b200.system import lambda_table, site_tables
from paper_2410_01754_b200.waterbox import generate_water_box

system, lam, _ = generate_water_box(3000, 4, seed=0)
for precision in ("double", "single"):
    s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=3, precision=precision))
    r = hi_energy_and_forces(system, lam.values, solver=s, spatial_forces=True)
    plan = s.plan
    plan.set_sites(*site_tables(system))
    lt, nl = lambda_table(system, lam.values)
    e, f, lf = np.empty(1), np.empty((system.num_particles, 3)), np.empty((4, 4))
    plan.step(system.positions, system.charges, lt, nl, mode=_native.MODE_HI, energy=e, forces=f, lambda_forces=lf)
    print(precision, r.energy, e[0])

# device-resident step (the benchmarked call: early HI side stream, positions
# copy inside k_wrap_cell, fused step tail, step graph on the repeat) at depth
# 5, where the leaf scan uses the look-back kernel and the big M2M / L2L
# levels the 64-column tensor-core tiles
import torch  # noqa: E402

system, lam, _ = generate_water_box(20000, 8, seed=1)
s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=5, precision="single"))
plan = s.plan
plan.set_sites(*site_tables(system))
lt, nl = lambda_table(system, lam.values)
dev = torch.device("cuda", 0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
d_pos, d_q, d_lam, d_nl = d(system.positions), d(system.charges), d(lt), d(nl)
d_e = torch.empty(1, dtype=torch.float64, device=dev)
d_f = torch.empty((system.num_particles, 3), dtype=torch.float64, device=dev)
d_lf = torch.empty((len(system.sites), 4), dtype=torch.float64, device=dev)
for _ in range(3):
    plan.step(d_pos, d_q, d_lam, d_nl, mode=_native.MODE_HI, on_device=True, energy=d_e, forces=d_f,
              lambda_forces=d_lf)
torch.cuda.synchronize()
print("device step", float(d_e[0]))
