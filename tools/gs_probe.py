"""Development probe: device time of one Gauss-Seidel launch per level (CUDA events)."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K

for k in [int(a) for a in sys.argv[1:]] or [0, 5]:
    h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
    D = h.dag_depth()
    M = h.num_macros()
    for l in range(1, 8):
        n = 1 << l
        u = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
        b = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
        for sweeps in (1, 2):
            s.gauss_seidel(u, b, sweeps)
            reps = 5
            t0 = time.perf_counter()
            for _ in range(reps):
                s.gauss_seidel(u, b, sweeps)
            dt = (time.perf_counter() - t0) / reps
            print(f"k={k} M={M} D={D} level={l} n={n} sweeps={sweeps}: {dt*1e6:9.1f} us  "
                  f"per DAG-step {dt*1e9/(sweeps*D*(2*n+1)):7.1f} ns", flush=True)
