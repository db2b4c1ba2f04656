"""Development probe: bandwidth of the level-wide kernels at large levels (CUDA events)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
L = int(sys.argv[2]) if len(sys.argv) > 2 else 10
t0 = time.time()
h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), L)
print(f"build {time.time()-t0:.1f}s", flush=True)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
N = h.level_size(L)
dofs = h.dof_count(L)
x = K.GridFunction(h, L, np.random.rand(N))
b = K.GridFunction(h, L, np.random.rand(N))
y = K.GridFunction(h, L)
xc = K.GridFunction(h, L - 1, np.random.rand(h.level_size(L - 1)))


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps


peak = 6469.3
for name, fn, bytes_per in [("apply", lambda: s.apply(K.STIFFNESS, x, y), 16 * dofs),
                            ("residual", lambda: s.residual(x, b, y), 24 * dofs),
                            ("restrict", lambda: s.restrict_transpose(x, xc), 8 * dofs + 8 * h.dof_count(L - 1)),
                            ("prolong", lambda: s.prolongate(xc, x), 8 * dofs + 8 * h.dof_count(L - 1))]:
    dt = timeit(fn)
    print(f"{name:9s} L={L} dofs={dofs} {dt*1e3:8.3f} ms  {bytes_per/dt/1e9:8.1f} GB/s  {bytes_per/dt/1e9/peak*100:5.1f}% of HBM (incl. host sync)", flush=True)
