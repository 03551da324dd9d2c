#!/usr/bin/env python
"""Benchmark of one full FMM + HI electrostatics step (BASELINE.json metric).

Workload (BASELINE.json configs[2], the paper headline on one GPU): a
synthetic ~1M-atom TIP3P-like water box with 512 titratable 10-atom sites
(2 forms each), p = 10, depth 5, fp32 kernels (fp64 reductions).  One step =
tree rebuild from the step's positions + scale_charges + solve (potentials,
near/far/dipole, energies) + spatial forces + HI corrections + lambda-force
assembly.  The "plain FMM" step (same positions, same
blended charges, no lambda machinery) is timed alongside for the HI
overhead.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun (N > 1) the step is the slab-decomposed one
(paper_2410_01754_b200/distributed.py): one global water box
of N x 1M atoms (weak scaling, depth 5 for N <= 2 and 6 for N >= 4 so that
leaves keep ~15-30 atoms), 512 sites, each rank owning an x slab of leaves;
value = N 1M-atom units / max-over-ranks step time.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FMM+HI electrostatics steps/sec at 1M atoms/512 sites; HI overhead % vs FMM"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--atoms", type=int, default=1_000_000)
    ap.add_argument("--sites", type=int, default=512)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--depth", type=int, default=5)
    ap.add_argument("--precision", default="single", choices=["single", "double"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 collectives (gloo only for single-GPU functional checks)")
    return ap.parse_args()


# ------------------------------------------------------------- helpers ----
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_system(args, rank):
    from paper_2410_01754_b200.waterbox import generate_water_box

    cache = f"/tmp/lfmm_wb_{args.atoms}_{args.sites}_{args.seed + rank}.npz"
    if os.path.exists(cache):
        z = np.load(cache)
        from paper_2410_01754_b200.system import LambdaState, ParticleSystem, TitratableSite

        off = z["site_off"]
        sites = [TitratableSite(z["site_idx"][off[s]:off[s + 1]], z["site_forms"][s]) for s in range(len(off) - 1)]
        system = ParticleSystem(float(z["box"]), z["positions"], z["charges"], sites)
        lam = LambdaState(values=list(z["lams"][:, None]) if z["lams"].ndim == 1 else list(z["lams"]),
                          velocities=[np.zeros(1)] * len(sites), masses=[5.0] * len(sites))
        return system, lam
    n_sites = args.sites
    # waters removed around each site (~8.25 molecules) are compensated
    target = args.atoms + int(round(n_sites * (3 * 8.25 - 10)))
    system, lam, _ = generate_water_box(target, n_sites, forms_per_site=2, seed=args.seed + rank)
    try:
        off = np.concatenate([[0], np.cumsum([s.num_particles for s in system.sites])])
        np.savez(cache, box=system.box_length, positions=system.positions, charges=system.charges,
                 site_off=off, site_idx=np.concatenate([s.particle_indices for s in system.sites]),
                 site_forms=np.stack([s.form_charges for s in system.sites]),
                 lams=np.array([v[0] for v in lam.values]))
    except OSError:
        pass
    return system, lam


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def pair_count(leaf_start, depth):
    """Exact ordered P2P pair count: sum_b sum_t n_b n_nb(b,t) - N."""
    n = 2 ** depth
    cnt = np.diff(leaf_start).astype(np.float64)
    g = np.arange(n ** 3)
    gx, gy, gz = g // (n * n), (g // n) % n, g % n
    tot = 0.0
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                nb = (((gx + dx) % n) * n + (gy + dy) % n) * n + (gz + dz) % n
                tot += float(np.dot(cnt, cnt[nb]))
    return tot - cnt.sum()


def algorithmic_work(p, depth, n_atoms, pairs, n_sites, ns=10, nf=2):
    """Closed-form work per step."""
    nc = (p + 1) ** 2
    boxes = sum(8 ** l for l in range(1, depth + 1))
    t_m2l = 189 * boxes
    w = {
        "p2p": {"flop": 20.0 * pairs, "bytes": 2 * 16.0 * n_atoms},
        "m2l": {"flop": 2.0 * nc * nc * t_m2l, "bytes": 2.0 * 4 * nc * boxes},
        "l2l": {"flop": 2.0 * nc * nc * boxes, "bytes": 3.0 * 4 * nc * boxes},
        "m2m": {"flop": 2.0 * nc * nc * boxes, "bytes": 4.0 * nc * boxes * 2},
        "p2m": {"flop": 8.0 * nc * n_atoms, "bytes": 16.0 * n_atoms + 4.0 * nc * 8 ** depth},
        "l2p": {"flop": 16.0 * nc * n_atoms, "bytes": 16.0 * n_atoms + 4.0 * nc * 8 ** depth + 16.0 * n_atoms},
        "hi": {"flop": n_sites * (20.0 * 27 * ns * ns + nf * (2.0 * nc * nc + 8 * ns * nc)), "bytes": 0.0},
        "t_m2l": t_m2l,
    }
    return w


# ------------------------------------------------- our arm, N > 1 ----
def run_distributed(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    dev_index = local if args.dist_backend == "nccl" else 0
    torch.cuda.set_device(dev_index)
    dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", dev_index)
    from paper_2410_01754_b200 import _native
    from paper_2410_01754_b200.distributed import DistributedSolver, TorchComm
    from paper_2410_01754_b200.fmm.solver import SolverConfig
    from paper_2410_01754_b200.system import lambda_table, site_tables

    depth = args.depth + (1 if world >= 4 else 0)
    gargs = argparse.Namespace(**vars(args))
    gargs.atoms = args.atoms * world
    # one global system (same seed on every rank); rank 0 generates and caches it first
    if rank == 0:
        system, lam_state = load_system(gargs, 0)
    dist.barrier()
    if rank != 0:
        system, lam_state = load_system(gargs, 0)
    n = system.num_particles
    cfg = SolverConfig(p=args.p, depth=depth, precision=args.precision)
    comm = TorchComm()
    solver = DistributedSolver(system.box_length, cfg, comm=comm)
    tables = site_tables(system)
    lam, nl = lambda_table(system, lam_state.values)
    s = len(system.sites)
    # each rank holds only the atoms of its own slab (global ids); the
    # boundary planes come from the neighbour ranks every step
    from paper_2410_01754_b200.distributed import leaf_x, wrap

    lx = leaf_x(wrap(system.positions, system.box_length), system.box_length, depth)
    own = np.flatnonzero((lx >= solver.x0) & (lx < solver.x1))
    d_pos = torch.from_numpy(np.ascontiguousarray(system.positions[own])).to(dev)
    d_q = torch.from_numpy(np.ascontiguousarray(system.charges[own])).to(dev)
    d_gid = torch.from_numpy(own.astype(np.int64)).to(dev)
    d_lam = torch.from_numpy(lam).to(dev)
    d_nl = torch.from_numpy(nl).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step_dev(plain=False):
        if plain:
            return solver.step_owned(d_pos, d_qt, d_gid)
        return solver.step_owned(d_pos, d_q, d_gid, d_lam, d_nl, sites=tables, n_global=n)

    # plain FMM: the same blended charges, no lambda machinery
    from paper_2410_01754_b200.system import scale_charges
    from paper_2410_01754_b200.weights import expand_weights

    qt = scale_charges(system, [expand_weights(np.asarray(v).reshape(-1)) for v in lam_state.values])
    d_qt = torch.from_numpy(np.ascontiguousarray(qt[own])).to(dev)
    out = step_dev()  # builds the plan

    def timed(fn, k):
        times = []
        for _ in range(k):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return times

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        step_dev()
        step_dev(plain=True)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = solver.plan.launch_count()
    clk = ClockSampler(dev_index).__enter__()
    t_full = timed(step_dev, args.steps)
    launches = (solver.plan.launch_count() - l0) // args.steps
    t_plain = timed(lambda: step_dev(plain=True), args.steps)
    torch.cuda.synchronize()
    dist.barrier()
    ms_full = max_over_ranks(sum(t_full) / len(t_full))
    ms_plain = max_over_ranks(sum(t_plain) / len(t_plain))

    # e2e: host inputs copied to the device every step, owned forces and lambda forces back
    h_pos = torch.from_numpy(np.ascontiguousarray(system.positions[own])).pin_memory()
    h_q = torch.from_numpy(np.ascontiguousarray(system.charges[own])).pin_memory()

    def step_host():
        d_pos.copy_(h_pos, non_blocking=True)
        d_q.copy_(h_q, non_blocking=True)
        o = step_dev()
        f = o["forces"].to("cpu", non_blocking=True)
        lf = o["lambda_forces"].to("cpu", non_blocking=True) if s else None
        torch.cuda.current_stream().synchronize()
        return f, lf

    step_host()
    dist.barrier()
    t_e2e = timed(step_host, args.steps)
    clk.__exit__(None, None, None)
    ms_e2e = max_over_ranks(sum(t_e2e) / len(t_e2e))
    n_own = int(out["owned"].numel())
    h2d = len(own) * 3 * 8 + len(own) * 8
    d2h = n_own * 3 * 8 + s * 4 * 8

    solver.plan.profile(True)
    kprof = max(3, min(args.steps, 10))
    for _ in range(kprof):
        step_dev()
    torch.cuda.synchronize()
    stages = solver.plan.stage_times()
    solver.plan.profile(False)
    stage_rows = {}
    for name, (ms_tot, cnt) in stages.items():
        if cnt == 0 or name == "setup":
            continue
        stage_rows[name] = {"ms": round(ms_tot / kprof, 4), "launches_per_step": cnt // kprof}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(world * 1000.0 / ms_full, 3), "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_full, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.precision == "single" else "f64",
            "data": "synthetic",
            "config": {"workload": f"C5-style weak scaling: one ~{n} atom water box ({args.atoms} per GPU), {s} "
                                   f"sites x 2 forms, p={args.p}, depth={depth}, x-slab octree decomposition over "
                                   f"{world} GPUs (distributed.py); value in 1M-atom step units",
                       "atoms": n, "sites": s, "p": args.p, "depth": depth,
                       "parallelism": f"slab decomposition x{world}, {args.dist_backend}",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "hi_overhead_pct": round(100.0 * (ms_full / ms_plain - 1.0), 2),
            "plain_fmm_ms_per_step": round(ms_plain, 4),
            "e2e": {"value": round(world * 1000.0 / ms_e2e, 3), "unit": "steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e, 4)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "roofline": None,
            "stages_rank0": stage_rows,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


# ----------------------------------------------------------- our arm ----
def run_ours(args):
    if dist_env()[1] > 1:
        return run_distributed(args)
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    from paper_2410_01754_b200 import _native
    from paper_2410_01754_b200.fmm.solver import PeriodicSolver, SolverConfig
    from paper_2410_01754_b200.system import lambda_table, site_tables

    system, lam_state = load_system(args, rank)
    n = system.num_particles
    cfg = SolverConfig(p=args.p, depth=args.depth, precision=args.precision)
    solver = PeriodicSolver(system.positions, system.box_length, cfg)
    plan = solver.plan
    tables = site_tables(system)
    plan.set_sites(*tables)
    lam, nl = lambda_table(system, lam_state.values)
    stream = torch.cuda.Stream(device=dev)
    plan.set_stream(stream.cuda_stream)
    s = len(system.sites)

    # device-resident inputs (value) -----------------------------------
    d_pos = torch.from_numpy(np.ascontiguousarray(system.positions)).to(dev)
    d_q = torch.from_numpy(np.ascontiguousarray(system.charges)).to(dev)
    d_lam = torch.from_numpy(np.ascontiguousarray(lam)).to(dev)
    d_nl = torch.from_numpy(np.ascontiguousarray(nl)).to(dev)
    d_e = torch.empty(1, dtype=torch.float64, device=dev)
    d_f = torch.empty((n, 3), dtype=torch.float64, device=dev)
    d_lf = torch.empty((s, 4), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # plain FMM charges: the same blended charges, no lambda machinery
    qt = plan.scale_charges(system.charges, lam, nl)
    d_qt = torch.from_numpy(qt).to(dev)

    def step_dev(plain=False):
        plan.step(d_pos, d_qt if plain else d_q, None if plain else d_lam, None if plain else d_nl,
                  mode=_native.MODE_HI, plain=plain, on_device=True, energy=d_e, forces=d_f, lambda_forces=d_lf)

    def timed(fn, k, flush_l2=True):
        times = []
        for _ in range(k):
            if flush_l2:
                with torch.cuda.stream(stream):
                    flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return times

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up
    for _ in range(max(3, args.warmup)):
        step_dev()
        step_dev(plain=True)
    torch.cuda.synchronize()

    # timed: full step, device-resident inputs
    l0 = plan.launch_count()
    barrier()
    clk = ClockSampler(local).__enter__()
    t_full = timed(step_dev, args.steps)
    barrier()
    launches = (plan.launch_count() - l0) // args.steps
    t_plain = timed(lambda: step_dev(plain=True), args.steps)
    ms_full = max_over_ranks(sum(t_full) / len(t_full))
    ms_plain = max_over_ranks(sum(t_plain) / len(t_plain))
    # plan reuse: tree frozen (positions not passed), as PeriodicSolver
    # holds one set of positions (solver.py:328-343)
    t_reuse = timed(lambda: plan.step(None, d_q, d_lam, d_nl, mode=_native.MODE_HI, plain=False, on_device=True,
                                      energy=d_e, forces=d_f, lambda_forces=d_lf), args.steps)
    ms_reuse = max_over_ranks(sum(t_reuse) / len(t_reuse))

    # e2e through the C-ABI with pinned host buffers
    h_pos = torch.from_numpy(np.ascontiguousarray(system.positions)).pin_memory()
    h_q = torch.from_numpy(np.ascontiguousarray(system.charges)).pin_memory()
    h_lam = torch.from_numpy(np.ascontiguousarray(lam)).pin_memory()
    h_nl = torch.from_numpy(np.ascontiguousarray(nl)).pin_memory()
    h_e = torch.empty(1, dtype=torch.float64).pin_memory()
    h_f = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    h_lf = torch.empty((s, 4), dtype=torch.float64).pin_memory()

    def step_host():
        plan.step(h_pos, h_q, h_lam, h_nl, mode=_native.MODE_HI, plain=False, on_device=False, energy=h_e,
                  forces=h_f, lambda_forces=h_lf)

    for _ in range(2):
        step_host()
    barrier()
    t_e2e = timed(step_host, args.steps)
    barrier()
    clk.__exit__(None, None, None)
    ms_e2e = max_over_ranks(sum(t_e2e) / len(t_e2e))
    h2d = n * 3 * 8 + n * 8 + s * 4 * 8 + s * 4
    d2h = 8 + n * 3 * 8 + s * 4 * 8
    # the PCIe rates of this box for the same pinned buffers (plain copies,
    # CUDA events): device step + host->device + device->host bytes at
    # these rates is the serial bound the e2e step is compared with
    def copy_rate(dst, src, reps=10):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        return src.numel() * src.element_size() * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    h2d_gbs = copy_rate(d_pos, h_pos)
    d2h_gbs = copy_rate(h_f, d_f)
    e2e_bound = ms_full + h2d / (h2d_gbs * 1e6) + d2h / (d2h_gbs * 1e6)

    # per-stage breakdown (separate profiled pass, CUDA events per launch)
    plan.profile(True)
    kprof = max(3, min(args.steps, 10))
    for _ in range(kprof):
        step_dev()
    stages = plan.stage_times()
    plan.profile(False)

    perm, inv, leaf, start, _ = plan.export_tree()
    pairs = pair_count(start, args.depth)
    work = algorithmic_work(args.p, args.depth, n, pairs, s)
    peaks, peak_kind = measured_peaks()
    stage_rows = {}
    step_ms = sum(v[0] for v in stages.values()) / kprof
    for name, (ms_tot, cnt) in stages.items():
        if cnt == 0 or name in ("setup",):
            continue
        ms = ms_tot / kprof
        row = {"ms": round(ms, 4), "launches_per_step": cnt // kprof,
               "share": round(ms / step_ms, 4) if step_ms else None}
        if name in work and isinstance(work[name], dict):
            fl = work[name]["flop"]
            row["algorithmic_gflop"] = round(fl / 1e9, 3)
            row["achieved_tflops"] = round(fl / (ms * 1e-3) / 1e12, 3) if ms > 0 else None
        stage_rows[name] = row
    # Roofline of the dominant tensor-core kernel, k_m2l_halo ("m2l" stage =
    # that launch alone; its absmax/pack passes are "m2l_pack").  Algorithmic
    # work = 2 (p+1)^4 flop per M2L translation (dense real-packed operator,
    # SURVEY.md 8d) x 189 sum_l 8^l translations per launch; the kernel issues
    # 3 fp16 products per term on 128x128 padded operators, counted separately
    # as "issued_tflops".  Peak = measured dense bf16 (= fp16) tensor rate.
    peaks, peak_kind = measured_peaks()
    m2l_ms = stage_rows.get("m2l", {}).get("ms", 0.0)
    fl = work["m2l"]["flop"]
    achieved = fl / (m2l_ms * 1e-3) / 1e12 if m2l_ms > 0 else 0.0
    t_m2l = work["t_m2l"]
    issued = 3 * 2.0 * 128 * 128 * t_m2l
    # ncu DRAM bytes of one M2L launch, captured on this workload (C3 fp32
    # only: the profile is static)
    traffic = None
    if (args.atoms, args.sites, args.p, args.depth, args.precision) == (1_000_000, 512, 10, 5, "single"):
        try:
            with open(os.path.join(ROOT, "profiles", "r02_final_ncu_full.json")) as fh:
                k = next(k for k in json.load(fh)["kernels"] if "k_m2l_halo" in k["kernel"])
            traffic = int(round((float(k["dram__bytes_read.sum"]) + float(k["dram__bytes_write.sum"])) * 1e6))
        except (OSError, StopIteration, KeyError, ValueError):
            pass
    roofline = {
        "kernel": "k_m2l_halo (M2L, tcgen05 kind::f16 3-product split)", "bound": "tensor",
        "achieved": round(achieved, 3), "peak": peaks.get("bf16_tflops"), "unit": "TFLOP/s",
        "frac": round(achieved / peaks.get("bf16_tflops", 1.0), 5), "traffic": traffic,
        "peak_source": f"{peak_kind} dense bf16 tensor rate (MEASURED_PEAKS.json; fp16 runs at the same rate)",
        "algorithmic": "2*(p+1)^4 flop per M2L translation x 189*sum_l 8^l translations per launch "
                       f"({t_m2l} translations)",
        "issued_tflops": round(issued / (m2l_ms * 1e-3) / 1e12, 3) if m2l_ms > 0 else None,
        "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of one launch "
                          "(profiles/r02_final_ncu_full.json)",
    }
    p2p_ms = stage_rows.get("p2p", {}).get("ms", 0.0)
    fp32_pipe = 62.2  # TFLOP/s, FFMA microbenchmark on this pool (profiles/r01_pipe_peaks.txt)
    p2p_tf = work["p2p"]["flop"] / (p2p_ms * 1e-3) / 1e12 if p2p_ms > 0 else 0.0
    roofline_p2p = {"kernel": "k_p2p2 (near field, packed f32x2)", "bound": "fp32 pipe",
                    "achieved": round(p2p_tf, 3), "peak": fp32_pipe, "unit": "TFLOP/s",
                    "frac": round(p2p_tf / fp32_pipe, 4),
                    "algorithmic": "20 flop per ordered pair (potential + gradient), exact pair count"}

    # the precision-matched (fp64, the reference's complex128 arithmetic) step
    # on the same system and call, with its own clock record
    fp64 = None
    if args.precision == "single":
        s64 = PeriodicSolver(system.positions, system.box_length,
                             SolverConfig(p=args.p, depth=args.depth, precision="double"))
        p64 = s64.plan
        p64.set_sites(*tables)
        p64.set_stream(stream.cuda_stream)

        def step64():
            p64.step(d_pos, d_q, d_lam, d_nl, mode=_native.MODE_HI, plain=False, on_device=True, energy=d_e,
                     forces=d_f, lambda_forces=d_lf)

        for _ in range(max(3, args.warmup)):
            step64()
        torch.cuda.synchronize()
        barrier()
        clk64 = ClockSampler(local).__enter__()
        t64 = timed(step64, args.steps)
        clk64.__exit__(None, None, None)
        ms64 = max_over_ranks(sum(t64) / len(t64))
        fp64 = {"value": round(world * 1000.0 / ms64, 3), "unit": "steps/s", "ms_per_step": round(ms64, 4),
                "dtype": "f64", "clocks": clk64.summary(),
                "what": "the same full step (tree rebuild + scale + solve + forces + HI + lambda forces) on fp64 "
                        "kernels (M2L on DMMA), device-resident inputs, L2 flushed between steps"}
        del s64, p64

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu = cpu_sample(system, lam_state, args)

    value = world * 1000.0 / ms_full
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_full, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "single" else "f64", "data": "synthetic",
        "config": {"workload": f"C3: ~{n} atom TIP3P-like water box, {s} titratable sites x 2 forms, p={args.p}, "
                               f"depth={args.depth}, {args.precision}; full step = tree rebuild + scale_charges + "
                               f"solve + spatial forces + HI corrections + lambda forces",
                   "atoms": n, "sites": s, "p": args.p, "depth": args.depth,
                   "parallelism": "replicas (one independent system per rank)" if world > 1 else "single GPU",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "hi_overhead_pct": round(100.0 * (ms_full / ms_plain - 1.0), 2),
        "plain_fmm_ms_per_step": round(ms_plain, 4),
        "plan_reuse_ms_per_step": round(ms_reuse, 4),
        "e2e": {"value": round(world * 1000.0 / ms_e2e, 3), "unit": "steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e, 4),
                "pcie_h2d_gbs": round(h2d_gbs, 1), "pcie_d2h_gbs": round(d2h_gbs, 1),
                "serial_bound_ms": round(e2e_bound, 4)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": roofline,
        "roofline_p2p": roofline_p2p,
        "stages": stage_rows,
        "p2p_pairs": pairs,
        "cpu_baseline": cpu,
        "fp64_step": fp64,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# ---------------------------------------------------- CPU (oracle) arm ----
def _thread_env(threads):
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[k] = str(threads)


def _oracle_inputs(system, lam_state, args):
    from oracle import lfmm_oracle as orc

    cfg = orc.default_config(p=args.p, depth=args.depth)
    sites = [(s.particle_indices, s.form_charges) for s in system.sites]
    lams = [np.asarray(v) for v in lam_state.values]
    return orc, cfg, sites, lams


def _cpu_worker(argv, threads, n_warm, n_timed, barrier, out_q):
    """One CPU worker process: full oracle steps (oracle/lfmm_oracle.full_step,
    nothing sampled), n_warm untimed, then n_timed after the start barrier."""
    _thread_env(threads)
    args = argparse.Namespace(**argv)
    system, lam_state = load_system(args, 0)
    orc, cfg, sites, lams = _oracle_inputs(system, lam_state, args)
    orc.lattice_matrix(cfg, system.box_length)  # per-process cache (lru_cache in the reference)
    tiny = system.positions[:64]  # numba JIT of the P2P loops outside any step
    orc.full_step(tiny, system.charges[:64], system.box_length, [], [], orc.default_config(p=2, depth=0),
                  time.perf_counter)
    for _ in range(n_warm):
        orc.full_step(system.positions, system.charges, system.box_length, sites, lams, cfg, time.perf_counter)
    barrier.wait()
    for _ in range(n_timed):
        t, parts, _ = orc.full_step(system.positions, system.charges, system.box_length, sites, lams, cfg,
                                    time.perf_counter)
        out_q.put((t, parts))
    out_q.put(None)


def cpu_throughput(args, steps, warmup):
    """Full oracle steps of the workload on the host cores: `steps` complete
    steps (tree + scale + solve + spatial forces + HI + lambda forces, no
    sampling or extrapolation) run by P concurrent worker processes of T
    threads (P * T = host cores), warm-up steps first; steps/s = steps /
    wall time of the timed region."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    threads = 2 if cores >= 4 else 1
    workers = max(1, min(steps, cores // threads))
    share = lambda n, w: n // workers + (1 if w < n % workers else 0)  # noqa: E731
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(workers + 1)
    out_q = ctx.Queue()
    argv = vars(args).copy()
    procs = [ctx.Process(target=_cpu_worker, args=(argv, threads, share(warmup, w), share(steps, w), barrier, out_q))
             for w in range(workers)]
    # the spawned interpreters import numpy before the worker function runs:
    # their BLAS / OpenMP / numba pools are sized from the inherited environment
    saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS",
                                            "NUMBA_NUM_THREADS")}
    _thread_env(threads)
    try:
        for p in procs:
            p.start()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    barrier.wait()
    t0 = time.perf_counter()
    lat, parts, done = [], [], 0
    while done < workers:
        item = out_q.get()
        if item is None:
            done += 1
        else:
            lat.append(item[0])
            parts.append(item[1])
    wall = time.perf_counter() - t0
    for p in procs:
        p.join()
    mean_parts = {k: round(statistics.mean(pp[k] for pp in parts), 2) for k in parts[0]}
    return {"value": round(len(lat) / wall, 6), "unit": "steps/s", "cores": workers * threads, "kind": "port",
            "sample": f"{len(lat)} complete C3 steps (oracle/lfmm_oracle.full_step: tree + scale_charges + solve "
                      f"with spatial forces + HI corrections + lambda forces + HI site forces; nothing sampled or "
                      f"extrapolated) by {workers} concurrent worker processes x {threads} threads; serial numba "
                      f"P2P as the reference's (solver.py:164-195), numpy complex128 + OpenBLAS elsewhere",
            "wall_s": round(wall, 2), "step_latency_s": round(statistics.median(lat), 2),
            "parts_s": mean_parts}


def cpu_sample(system, lam_state, args):
    """Our arm's cpu_baseline: one complete oracle step on rank 0 with every
    host thread (latency; nothing sampled)."""
    _thread_env(os.cpu_count() or 1)
    orc, cfg, sites, lams = _oracle_inputs(system, lam_state, args)
    orc.lattice_matrix(cfg, system.box_length)
    t, parts, _ = orc.full_step(system.positions, system.charges, system.box_length, sites, lams, cfg,
                                time.perf_counter)
    return {"value": round(1.0 / t, 6), "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
            "sample": "one complete C3 step (oracle/lfmm_oracle.full_step, nothing sampled), one process, numpy / "
                      "OpenBLAS on every host thread, serial numba P2P as the reference's",
            "s_per_step": round(t, 2), "parts_s": {k: round(v, 2) for k, v in parts.items()}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    system, lam_state = load_system(args, 0)  # generate + cache once for the workers
    base = cpu_throughput(args, args.steps, args.warmup)
    t = 1.0 / base["value"]
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000 * t, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C3: ~{system.num_particles} atom water box, {len(system.sites)} sites, "
                                   f"p={args.p}, depth={args.depth}; oracle port on the host cores",
                       "atoms": system.num_particles, "sites": len(system.sites), "p": args.p, "depth": args.depth},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
