"""Per-CTA timing of k_m2l_halo from the profiling build (make prof):
LFMM_LIB=paper_2410_01754_b200/_lib/liblfmm_prof.so python tools/hm_prof.py"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("LFMM_LIB", os.path.join(ROOT, "paper_2410_01754_b200/_lib/liblfmm_prof.so"))
os.environ["LFMM_FAR"] = "serial"  # one k_m2l_halo launch (CTA index = job index)
sys.path.insert(0, ROOT)
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig, _native
from paper_2410_01754_b200.waterbox import generate_water_box

depth = 5
system, lam, _ = generate_water_box(1_000_000, 8, seed=4)
s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=depth, precision="single"))
for _ in range(3):
    s.solve(system.charges)
lib = _native.lib()
buf = np.zeros((8192, 8), np.uint64)
lib.lfmm_debug_hm_prof.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert lib.lfmm_debug_hm_prof(buf.ctypes.data, 8192) == 0
# job list (plan_halo_jobs)
jobs = []
for l in range(depth, 0, -1):
    h = 1 << (l - 1); Z = h + 2; S = Z * Z + Z + 1; last = h * S
    G = 4 if l >= 4 else 8
    t0 = S
    while t0 <= last:
        N = min(256, ((last + 1 - t0) + 15) // 16 * 16)
        for tc in range(8):
            for g in range(G):
                jobs.append((l, N, tc, g))
        t0 += 256
# plan_halo_jobs order: levels >= depth-1 first, big N first within a group
ls = depth - 1 if depth >= 3 else 1
jobs = sorted(jobs, key=lambda j: (0 if j[0] >= ls else 1, -j[1]))
nj = len(jobs)
b = buf[:nj].astype(np.float64)
t0 = b[:, 0].min()
start = (b[:, 0] - t0) / 1e3
end = (b[:, 1] - t0) / 1e3
mmaend = (b[:, 6] - t0) / 1e3
dur = end - start
print("jobs %d  kernel span %.1f us" % (nj, end.max()))
clk = 1.9e3  # cycles per us (approx)
for key in sorted(set((j[0], j[1]) for j in jobs), reverse=True):
    sel = np.array([(j[0], j[1]) == key for j in jobs])
    print("level %d N=%3d: %4d jobs  dur %.1f us  mma-issue %.1f us  tail(epi) %.1f us  wait halo %.1f acc %.1f A %.1f us  terms %.0f" % (
        key[0], key[1], sel.sum(), dur[sel].mean(), (mmaend - start)[sel].mean(), (end - mmaend)[sel].mean(),
        b[sel, 2].mean() / clk, b[sel, 3].mean() / clk, b[sel, 4].mean() / clk, b[sel, 5].mean()))
sm = b[:, 7].astype(int)
busy = np.zeros(148)
for i in range(nj):
    busy[sm[i]] += dur[i]
print("per-SM busy: min %.1f max %.1f mean %.1f us; start of last job %.1f us" % (busy.min(), busy.max(), busy.mean(), start.max()))
order = np.argsort(start)
print("first 5 starts", start[order[:5]], "last 5 ends", np.sort(end)[-5:])
