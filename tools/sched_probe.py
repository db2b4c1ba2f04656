"""Development probe: the static-schedule smoother on small cfg2 levels (CUDA events)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
st = torch.cuda.ExternalStream(s.stream())
for l in range(1, 6):
    u = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
    b = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
    s.interface_sync(u, K.SYNC_REPLACE)
    s.interface_sync(b, K.SYNC_REPLACE)
    s.gauss_seidel(u, b, 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(10):
        K._check(K.lib().klref_gauss_seidel(s.ptr, u.ptr, b.ptr, 2))
    e1.record(st)
    torch.cuda.synchronize()
    print(f"k={k} level={l}: {e0.elapsed_time(e1) * 100:.1f} us per 2-sweep call", flush=True)
