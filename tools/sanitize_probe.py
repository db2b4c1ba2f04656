"""Development probe for compute-sanitizer: the cross-CTA flag protocols of the
smoothers on small cases (2-d pipelined / static-schedule / macro-DAG kernels,
3-d cooperative multicolour kernel) and one FMG + estimate."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np

from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube

which = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)
if which in ("all", "2d"):
    h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", "cfg2_k3.mesh")), 5)
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
    for l in (2, 4, 5):  # static schedule (small), pipelined (n >= 16)
        u = K.GridFunction(h, l, rng.random(h.level_size(l)))
        b = K.GridFunction(h, l, rng.random(h.level_size(l)))
        s.interface_sync(u, K.SYNC_REPLACE)
        s.interface_sync(b, K.SYNC_REPLACE)
        s.gauss_seidel(u, b, 2)
    s.fmg()
    rep = s.error_estimate(1, K.UNSCALED)
    print("2d ok", rep.eta)
if which in ("all", "3d"):
    h = K.GridHierarchy.build(kuhn_cube(2), 4)
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_SIN3D), K.SolverConfig(nu=2))
    s.fmg()
    rep = s.error_estimate(1, K.UNSCALED)
    print("3d ok", rep.eta)
