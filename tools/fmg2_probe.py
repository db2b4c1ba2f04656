"""Development probe: cfg2 FMG + estimator per AMR mesh with in-graph kernel probes."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch

from paper_2508_06049_b200 import klref as K

ks = [int(a) for a in sys.argv[1:]] or list(range(6))
tot = {}
for k in ks:
    h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
    s.set_profiling(True)
    for _ in range(2):
        s.fmg_enqueue(); s.error_estimate_enqueue(1); s.synchronize(); s.error_estimate_finish(1, 0)
    st = torch.cuda.ExternalStream(s.stream())
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.fmg_enqueue(); s.error_estimate_enqueue(1)
        e1.record(st)
        s.synchronize(); s.error_estimate_finish(1, 0)
        best = min(best, e0.elapsed_time(e1))
    line = f"k={k} macros={h.num_macros()} FMG+est {best:.3f} ms:"
    for kk in range(8):
        m_, n_, b_ = s.kernel_stats(kk)
        tot[kk] = tot.get(kk, 0.0) + m_
        line += f" {K.KERNEL_NAMES[kk]} {m_:.2f}"
    print(line, flush=True)
print("sum over meshes:", " ".join(f"{K.KERNEL_NAMES[kk]} {v:.2f}" for kk, v in tot.items()))
