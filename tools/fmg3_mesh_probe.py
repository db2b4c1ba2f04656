"""Development probe: 3-d FMG + estimate kernel breakdown on a mesh file (e.g. tests/golden/cfg4_k4.mesh)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch

from paper_2508_06049_b200 import klref as K

path, L = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 6
h = K.GridHierarchy.build(K.MacroMesh.read(path), L)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_GAUSS3D), K.SolverConfig(nu=2))
s.set_profiling(True)
for _ in range(2):
    s.fmg_enqueue(); s.error_estimate_enqueue(1); s.synchronize(); s.error_estimate_finish(1, 0)
st = torch.cuda.ExternalStream(s.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); s.fmg_enqueue(); s.error_estimate_enqueue(1); e1.record(st); s.synchronize(); s.error_estimate_finish(1, 0)
ms = e0.elapsed_time(e1)
print(f"{path}: macros {h.num_macros()} dofs {h.dof_count(L)} FMG+est {ms:.2f} ms -> {h.dof_count(L)/ms/1e6:.3f} GDoF/s")
for k in range(8):
    m_, n_, b_ = s.kernel_stats(k)
    if n_:
        print(f"  {K.KERNEL_NAMES[k]:14s} {m_:8.3f} ms {n_:5d} launches")
