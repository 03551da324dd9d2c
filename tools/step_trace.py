"""Timeline of one C3 lfmm_step (profiling build: make prof) with every stream
running concurrently: per launch (stage, start, end) in us from CUDA events
recorded on the launching stream.
LFMM_LIB=paper_2410_01754_b200/_lib/liblfmm_prof.so python tools/step_trace.py [depth]"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("LFMM_LIB", os.path.join(ROOT, "paper_2410_01754_b200/_lib/liblfmm_prof.so"))
sys.path.insert(0, ROOT)
import torch
from paper_2410_01754_b200 import PeriodicSolver, SolverConfig, _native
from paper_2410_01754_b200.system import lambda_table, site_tables
from paper_2410_01754_b200.waterbox import generate_water_box

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 5
system, lam, _ = generate_water_box(1_000_000, 512, seed=0)
s = PeriodicSolver(system.positions, system.box_length, SolverConfig(p=10, depth=depth, precision="single"))
plan = s.plan
plan.set_sites(*site_tables(system))
lt, nl = lambda_table(system, lam.values)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(device=dev)
plan.set_stream(st.cuda_stream)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
d_pos, d_q, d_lam, d_nl = d(system.positions), d(system.charges), d(lt), d(nl)
n = system.num_particles
d_e = torch.empty(1, dtype=torch.float64, device=dev)
d_f = torch.empty((n, 3), dtype=torch.float64, device=dev)
d_lf = torch.empty((len(system.sites), 4), dtype=torch.float64, device=dev)
lib = _native.lib()
lib.lfmm_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.lfmm_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
lib.lfmm_debug_trace_read.restype = ctypes.c_int64
step = lambda: plan.step(d_pos, d_q, d_lam, d_nl, mode=0, on_device=True, energy=d_e, forces=d_f,  # noqa: E731
                         lambda_forces=d_lf)
for _ in range(5):
    step()
torch.cuda.synchronize()
names = [lib.lfmm_stage_name(i).decode() for i in range(lib.lfmm_stage_count())]
for rep in range(2):
    assert lib.lfmm_debug_trace(plan.h, 1) == 0
    step()
    torch.cuda.synchronize()
    buf = np.zeros((4096, 3))
    k = lib.lfmm_debug_trace_read(plan.h, buf.ctypes.data, 4096)
    lib.lfmm_debug_trace(plan.h, 0)
rows = buf[:k]
order = np.argsort(rows[:, 1])
print("launches %d  span %.1f us" % (k, rows[:, 2].max() * 1e3))
for i in order:
    stg, a, b = rows[i]
    print("%-9s %8.1f %8.1f  %7.1f" % (names[int(stg)], a * 1e3, b * 1e3, (b - a) * 1e3))
