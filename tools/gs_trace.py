"""Development probe: per-step clocks of the smoother (debug build tools/libklref_dbg.so)."""
import ctypes as C
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["KLREF_LIB"] = os.path.join(REPO, "tools", "libklref_dbg.so")
sys.path.insert(0, REPO)
import numpy as np

from paper_2508_06049_b200 import klref as K

k, l = int(sys.argv[1]), int(sys.argv[2])
h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
u = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
b = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
n = 1 << l
tr = np.zeros(4 << 12, dtype=np.int64)
try:
    s.gauss_seidel(u, b, 1)
    s.gauss_seidel(u, b, 1)
finally:
    K.lib().klref_debug_gs_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong)), tr.size)
    print("check record", tr.reshape(4, -1)[3, 4000:4004])
tr = tr.reshape(4, 1 << 12)[:, : 2 * n + 1]
d_step = np.diff(tr[0])
print("n", n, "steps", 2 * n + 1)
print("boundary-warp cycles/step: median", np.median(d_step), "mean", d_step.mean())
print("load_pre cycles median", np.median(tr[1] - tr[0]), "relax cycles median", np.median(tr[2] - tr[1]),
      "barrier wait median", np.median(tr[0][1:] - tr[2][:-1]))
print("interior warp cycles/step median", np.median(np.diff(tr[3])))
print("means: ring", (tr[1]-tr[0]).mean(), "relax", (tr[2]-tr[1]).mean(), "to next", (tr[0][1:]-tr[2][:-1]).mean())
for t in range(min(100, n), min(106, 2 * n)):
    print(t, tr[0][t]-tr[0][min(100,n)], tr[1][t]-tr[0][min(100,n)], tr[2][t]-tr[0][min(100,n)], "interior", tr[3][t]-tr[0][min(100,n)])
