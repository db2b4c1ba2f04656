"""Development probe: Gauss-Seidel launches over several meshes/levels in one process.
args: k:l[:sweeps[:reps]] ..."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np

from paper_2508_06049_b200 import klref as K

hs = {}
for spec in sys.argv[1:]:
    parts = [int(v) for v in spec.split(":")]
    k, l = parts[0], parts[1]
    sweeps = parts[2] if len(parts) > 2 else 1
    reps = parts[3] if len(parts) > 3 else 1
    if k not in hs:
        h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
        hs[k] = (h, K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2)))
    h, s = hs[k]
    u = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
    b = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
    for _ in range(reps):
        s.gauss_seidel(u, b, sweeps)
    print("ok", spec, flush=True)
