"""Development probe: 3-d FMG + estimator timing with kernel probes (cfg3 / cfg5 shapes)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
L = int(sys.argv[2]) if len(sys.argv) > 2 else 6
prob = sys.argv[3] if len(sys.argv) > 3 else "sin3"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
t0 = time.time()
h = K.GridHierarchy.build(kuhn_cube(N), L)
t1 = time.time()
kind = {"sin3": K.PROBLEM_SIN3D, "series": K.PROBLEM_SERIES3D}[prob]
s = K.MultigridSolver(h, K.Problem(kind, series_coefficients() if prob == "series" else None), K.SolverConfig(nu=2))
t2 = time.time()
print(f"N={N} L={L} macros={h.num_macros()} dofs={h.dof_count(L)} build {t1-t0:.1f}s solver {t2-t1:.1f}s", flush=True)
s.set_profiling(True)
for _ in range(1 if reps == 1 else 2):
    s.fmg_enqueue(); s.error_estimate_enqueue(1); s.synchronize(); rep = s.error_estimate_finish(1, 0)
st = torch.cuda.ExternalStream(s.stream())
times = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.fmg_enqueue(); s.error_estimate_enqueue(1)
    e1.record(st)
    s.synchronize(); rep = s.error_estimate_finish(1, 0)
    times.append(e0.elapsed_time(e1))
ms = min(times)
dofs = h.dof_count(L)
print(f"FMG+est {ms:.3f} ms  -> {dofs/ms/1e6:.3f} GDoF/s   eta={rep.eta:.4e} theta={rep.conv_factor:.4f}")
names = K.KERNEL_NAMES
for kk in range(8):
    m_, n_, b_ = s.kernel_stats(kk)
    if n_:
        print(f"  {names[kk]:12s} {m_:9.3f} ms  {n_:5d} launches  alg {b_/(m_*1e-3)/1e9 if m_>0 else 0:8.1f} GB/s")
print("level-0 CG iterations (last call):", s.last_cg_iterations())
