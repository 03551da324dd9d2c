"""Per-CTA timing of the persistent k_m2l_halo from the profiling build
(make prof): LFMM_LIB=paper_2410_01754_b200/_lib/liblfmm_prof.so python tools/hm_prof.py
Records per CTA: start, end, issuer waits on halo / accumulator / A ring
(clock64 cycles summed over both issuers), terms issued, last MMA issue, SM."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("LFMM_LIB", os.path.join(ROOT, "paper_2410_01754_b200/_lib/liblfmm_prof.so"))
sys.path.insert(0, ROOT)
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig, _native
from paper_2410_01754_b200.waterbox import generate_water_box

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
system, lam, _ = generate_water_box(1_000_000, 8, seed=4)
s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=depth, precision="single"))
for _ in range(3):
    s.solve(system.charges)
lib = _native.lib()
buf = np.zeros((8192, 8), np.uint64)
lib.lfmm_debug_hm_prof.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert lib.lfmm_debug_hm_prof(buf.ctypes.data, 8192) == 0
ncta = int((buf[:, 1] > 0).sum())
b = buf[:ncta].astype(np.float64)
t0 = b[:, 0].min()
start, end, mmaend = (b[:, 0] - t0) / 1e3, (b[:, 1] - t0) / 1e3, (b[:, 6] - t0) / 1e3
clk = 1.965e3  # cycles per us at the boost clock
span = end - start
terms = b[:, 5]
tensor_us = terms * 3 * 135 / clk  # ~135 clk per N=256 kind::f16 MMA (B200)
print("CTAs %d  kernel span %.1f us  CTA span mean %.1f min %.1f max %.1f" % (ncta, end.max(), span.mean(), span.min(),
                                                                             span.max()))
print("per CTA: last MMA issue %.1f us before its end; terms %.0f (tensor work ~%.1f us at N=256)" % (
    (end - mmaend).mean(), terms.mean(), tensor_us.mean()))
print("issuer waits per CTA (sum of 2 issuers): halo %.1f  acc %.1f  A %.1f us" % (
    b[:, 2].mean() / clk, b[:, 3].mean() / clk, b[:, 4].mean() / clk))
