"""Debug: single-GPU step energy pieces vs the slab-decomposed step (2 ranks as threads)."""
import sys, threading
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2410_01754_b200 import _native, hi_energy_and_forces
from paper_2410_01754_b200.distributed import DistributedSolver, LocalComm
from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig
from paper_2410_01754_b200.system import lambda_table, site_tables
from paper_2410_01754_b200.waterbox import generate_water_box

system, lam, _ = generate_water_box(40_000, 24, seed=11)
for precision in ("double", "single"):
    cfg = SolverConfig(p=10, depth=4, precision=precision)
    s = PeriodicSolver(system.positions, system.box_length, cfg)
    r = hi_energy_and_forces(system, lam.values, solver=s)
    print(precision, "hi_energy_and_forces", r.energy, "solve", float(r.solve.energy), "offset", r.corrections.energy_offset())
    plan = s.plan
    plan.set_sites(*site_tables(system))
    lt, nl = lambda_table(system, lam.values)
    e = np.empty(1); f = np.empty((system.num_particles, 3)); lf = np.empty((24, 4))
    plan.step(system.positions, system.charges, lt, nl, mode=_native.MODE_HI, energy=e, forces=f, lambda_forces=lf)
    print(precision, "step", e[0])
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(system.positions).to(dev); q = torch.from_numpy(system.charges).to(dev)
    d_lam = torch.from_numpy(lt).to(dev); d_nl = torch.from_numpy(nl).to(dev)
    tables = site_tables(system)
    shared = LocalComm(2); outs = [None, None]
    def run(rank):
        torch.cuda.set_device(0)
        sv = DistributedSolver(system.box_length, cfg, comm=shared.for_rank(rank))
        outs[rank] = sv.step(pos, q, d_lam, d_nl, sites=tables)
        torch.cuda.synchronize()
    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    [t.start() for t in th]; [t.join() for t in th]
    for o in outs:
        print(precision, "dist", o["energy"], "solve", o["energy_solve"], "near", o["near_energy"], "far", o["far_energy"], "dip", o["dipole_energy"])
    print(precision, "single near/far/dip", float(r.solve.near_energy), float(r.solve.far_energy), float(r.solve.dipole_energy))
