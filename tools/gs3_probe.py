"""Development probe: 3-d smoother time per level (2 sweeps), Kuhn cube N^3, levels 1..L."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 6
only = int(sys.argv[3]) if len(sys.argv) > 3 else -1
h = K.GridHierarchy.build(kuhn_cube(N), L)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_ZERO), K.SolverConfig(nu=2))
st = torch.cuda.ExternalStream(s.stream())
rng = np.random.default_rng(0)
for l in range(1, L + 1):
    if only >= 0 and l != only:
        continue
    sz = h.level_size(l)
    u = K.GridFunction(h, l, rng.standard_normal(sz))
    b = K.GridFunction(h, l, rng.standard_normal(sz))
    s.gauss_seidel(u, b, 2)
    s.synchronize()
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.gauss_seidel(u, b, 2)
        e1.record(st)
        s.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = min(times)
    d = h.dof_count(l)
    print(f"level {l}: n={2**l} dofs={d} GS x2 {ms:.3f} ms  alg {48.0*d/(ms*1e-3)/1e9:8.1f} GB/s", flush=True)
