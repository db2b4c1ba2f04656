"""Development probe: host-side set-up cost per cfg2 AMR mesh (hierarchy build + upload, solver, first FMG = graph capture)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2508_06049_b200 import klref as K

K.lib()
import torch  # noqa: E402

torch.cuda.init()
tot = [0.0, 0.0, 0.0, 0.0]
for rep in range(2):
    for k in range(6):
        mesh = K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh"))
        t0 = time.perf_counter()
        h = K.GridHierarchy.build(mesh, 7)
        t1 = time.perf_counter()
        s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
        t2 = time.perf_counter()
        s.fmg_enqueue(); s.synchronize()
        t3 = time.perf_counter()
        s.fmg_enqueue(); s.synchronize()
        t4 = time.perf_counter()
        if rep == 1:
            print(f"k={k} macros={h.num_macros()}: hierarchy {1e3*(t1-t0):.1f} ms, solver {1e3*(t2-t1):.1f} ms, "
                  f"first fmg {1e3*(t3-t2):.1f} ms, second fmg {1e3*(t4-t3):.1f} ms", flush=True)
            for i, d in enumerate((t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
                tot[i] += d
print("totals (s): hierarchy %.3f solver %.3f first-fmg %.3f second-fmg %.3f" % tuple(tot))
