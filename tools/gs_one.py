"""Development probe: one Gauss-Seidel launch on one level of one cfg2 mesh (for ncu)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np

from paper_2508_06049_b200 import klref as K

k, l, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1
h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
u = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
b = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
for _ in range(reps):
    s.gauss_seidel(u, b, 1)
print("ok")
