"""Development probe: one 2-sweep pipelined smoother call on a cfg2 level (trace via KB_PIPE_TRACE)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np

from paper_2508_06049_b200 import klref as K

k, l = int(sys.argv[1]), int(sys.argv[2])
h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
u = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
b = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
s.interface_sync(u, K.SYNC_REPLACE)
s.interface_sync(b, K.SYNC_REPLACE)
s.gauss_seidel(u, b, 2)
s.synchronize()
