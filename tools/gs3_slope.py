"""Development probe: 3-d smoother time against the sweep count (slope = time per sweep without launch cost)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
h = K.GridHierarchy.build(kuhn_cube(N), L)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_ZERO), K.SolverConfig(nu=2))
st = torch.cuda.ExternalStream(s.stream())
rng = np.random.default_rng(0)
for l in range(1, L + 1):
    sz = h.level_size(l)
    u = K.GridFunction(h, l, rng.standard_normal(sz))
    b = K.GridFunction(h, l, rng.standard_normal(sz))
    res = []
    for sw in (1, 2, 11, 21):
        s.gauss_seidel(u, b, sw)
        s.synchronize()
        times = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s.gauss_seidel(u, b, sw)
            e1.record(st)
            s.synchronize()
            times.append(e0.elapsed_time(e1))
        res.append(min(times))
    print(f"level {l}: n={2**l} sweeps 1/2/11/21: " + " ".join(f"{t*1e3:.1f}" for t in res) +
          f" us   per sweep {(res[3]-res[2])*100:.2f} us, fixed {res[1]*1e3 - 2*(res[3]-res[2])*100:.1f} us", flush=True)
