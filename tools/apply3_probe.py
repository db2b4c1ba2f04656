"""Development probe: 3-d level kernels (apply, residual, restrict, prolong, GS) at
level L of a Kuhn N^3 mesh, CUDA-event timed on the solver stream."""
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
h = K.GridHierarchy.build(kuhn_cube(N), L)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_ZERO), K.SolverConfig(nu=2))
st = torch.cuda.ExternalStream(s.stream())
rng = np.random.default_rng(0)
sz = h.level_size(L)
d = h.dof_count(L)
dc = h.dof_count(L - 1)
x = K.GridFunction(h, L, rng.standard_normal(sz))
b = K.GridFunction(h, L, rng.standard_normal(sz))
y = h.create_function(L)
xc = K.GridFunction(h, L - 1, rng.standard_normal(h.level_size(L - 1)))


def timeit(fn, reps=5):
    fn()
    s.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        s.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for name, fn, nb in [("apply", lambda: s.apply(K.STIFFNESS, x, y), 16 * d),
                     ("residual", lambda: s.residual(x, b, y), 24 * d),
                     ("restrict", lambda: s.restrict_transpose(x, xc), 8 * d + 8 * dc),
                     ("prolong", lambda: s.prolongate(xc, x), 8 * d + 8 * dc),
                     ("gs x2", lambda: s.gauss_seidel(x, b, 2), 48 * d)]:
    ms = timeit(fn)
    print(f"{name:9s} L={L} dofs={d} {ms:8.3f} ms  alg {nb / ms / 1e6:8.1f} GB/s", flush=True)
