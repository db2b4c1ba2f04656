"""Development probe: 3-d FMG + estimator timing at Kuhn N^3, level L (CUDA events)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch

from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 6
h = K.GridHierarchy.build(kuhn_cube(N), L)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_SERIES3D, series_coefficients(7)), K.SolverConfig(nu=2))
st = torch.cuda.ExternalStream(s.stream())
s.fmg()
s.error_estimate(1, K.UNSCALED)
s.synchronize()
best = [1e30, 1e30]
for _ in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(st)
    s.fmg()
    e[1].record(st)
    rep = s.error_estimate(1, K.UNSCALED)
    e[2].record(st)
    s.synchronize()
    best = [min(best[0], e[0].elapsed_time(e[1])), min(best[1], e[1].elapsed_time(e[2]))]
print(f"N={N} L={L} dofs={h.dof_count(L)} fmg {best[0]:.3f} ms  estimate {best[1]:.3f} ms  eta={rep.eta:.12e}")
