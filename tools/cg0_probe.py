"""Development probe: level-0 CG of a cfg2 mesh, time per call and iterations."""
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
rng = np.random.default_rng(0)
b = K.GridFunction(h, 0, rng.random(h.level_size(0)))
s.interface_sync(b, K.SYNC_REPLACE)
for rep in range(3):
    u = K.GridFunction(h, 0, np.zeros(h.level_size(0)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.cg_level0(u, b)
    e1.record(st)
    s.synchronize()
    it = s.last_cg_iterations()
    ms = e0.elapsed_time(e1)
print(f"k={k}: level-0 dofs {h.dof_count(0)} copies {h.level_size(0)}: {ms*1e3:.1f} us, {it} iterations, {ms*1e3/max(it,1):.2f} us/iteration")
