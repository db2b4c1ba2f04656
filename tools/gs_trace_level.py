"""Development probe: per-item clocks of k_gs_level (debug build tools/libklref_dbg.so)."""
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
s.gauss_seidel(u, b, 1)
tr = np.zeros(4 << 12, dtype=np.int64)
K.lib().klref_debug_gs_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong)), tr.size)
tr = tr.reshape(4, -1)
it = tr[2][:4 * 40].reshape(-1, 4)
it = it[it[:, 0] > 0]
base = it[0, 0]
print("item: start, wait+bar, ghosts+bar, sweep+bar (cycles rel.)")
for r in it[:12]:
    print(r[0] - base, r[1] - r[0], r[2] - r[1], r[3] - r[2])
print("per-step cycles (group 0 boundary warp):", np.median(np.diff(tr[0][: 2 * (1 << l) + 1])))
