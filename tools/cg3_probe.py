"""Development probe: 3-d level-0 CG (iterations, time per call) on Kuhn N^3."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
h = K.GridHierarchy.build(kuhn_cube(N), 2)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_SERIES3D, series_coefficients(7)), K.SolverConfig(nu=2))
st = s.fmg()
print("fmg last cg iterations", s.last_cg_iterations())
b = K.GridFunction(h, 0, st.b(0))
stream = torch.cuda.ExternalStream(s.stream())
for rep in range(3):
    u = K.GridFunction(h, 0, np.zeros(h.level_size(0)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.cg_level0(u, b)
    e1.record(stream)
    s.synchronize()
    print(f"cg0 from zero: {s.last_cg_iterations()} iterations, {e0.elapsed_time(e1):.3f} ms")
