"""Secondary measurements of SURVEY.md §8d (single GPU), beside bench.py's
headline: C2 (100k atoms, 64 sites, depth 4) in fp32 and fp64, C3 in fp64,
C3 with the tree frozen (plan reuse), C4 (4096 sites), C3 at depth 4, C5's
8M-atom box (depth 6) on one GPU, and the reference's
HI-overhead definition t_corr / t_solve.  Device-resident inputs, L2 flushed
between steps, CUDA events on the plan's stream, mean of K steps after W
warm-ups.  Prints one JSON object."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(atoms, sites, depth, precision, steps=10, warmup=3, seed=0, reuse=False):
    import torch

    from paper_2410_01754_b200 import _native
    from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig
    from paper_2410_01754_b200.system import lambda_table, site_tables
    from paper_2410_01754_b200.waterbox import generate_water_box

    target = atoms + int(round(sites * (3 * 8.25 - 10)))
    t0 = time.time()
    system, lam_state, _ = generate_water_box(target, sites, forms_per_site=2, seed=seed)
    gen_s = time.time() - t0
    dev = torch.device("cuda", 0)
    solver = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=depth, precision=precision))
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
    d_lf = torch.empty((max(s, 1), 4), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    qt = plan.scale_charges(system.charges, lam, nl)
    d_qt = torch.from_numpy(qt).to(dev)

    def run(plain):
        plan.step(None if reuse else d_pos, d_qt if plain else d_q, None if plain else d_lam,
                  None if plain else d_nl, mode=_native.MODE_HI, plain=plain, on_device=True, energy=d_e,
                  forces=d_f, lambda_forces=d_lf)

    def timed(plain):
        for _ in range(warmup):
            run(plain)
        ts = []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run(plain)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.mean(ts))

    ms_full, ms_plain = timed(False), timed(True)
    plan.profile(True)
    for _ in range(5):
        run(False)
    st = plan.stage_times()
    plan.profile(False)
    t_corr = (st["hi"][0] + st["scale"][0]) / 5
    t_solve = sum(v[0] for k, v in st.items() if k not in ("hi", "scale", "setup")) / 5
    return {"atoms": n, "sites": s, "depth": depth, "precision": precision, "tree_frozen": reuse,
            "ms_per_step": round(ms_full, 4), "plain_fmm_ms": round(ms_plain, 4),
            "hi_overhead_pct": round(100 * (ms_full / ms_plain - 1), 2),
            "hi_overhead_ref_def_pct": round(100 * t_corr / t_solve, 2), "generate_s": round(gen_s, 1),
            "stages_ms": {k: round(v[0] / 5, 4) for k, v in st.items() if v[1]}}


def main():
    out = {"gpu": "B200 x1", "how": __doc__.split("\n\n")[0].replace("\n", " "), "runs": []}
    only = sys.argv[1:]  # optional run indices
    runs = (dict(atoms=100_000, sites=64, depth=4, precision="single"),
               dict(atoms=100_000, sites=64, depth=4, precision="double"),
               dict(atoms=1_000_000, sites=512, depth=5, precision="single", reuse=True),
               dict(atoms=1_000_000, sites=512, depth=5, precision="double"),
               dict(atoms=1_000_000, sites=4096, depth=5, precision="single"),
               dict(atoms=1_000_000, sites=512, depth=4, precision="single"),
               dict(atoms=8_000_000, sites=512, depth=6, precision="single"))
    for i, kw in enumerate(runs):
        if only and str(i) not in only:
            continue
        r = measure(**kw)
        print(json.dumps(r), flush=True)
        out["runs"].append(r)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
