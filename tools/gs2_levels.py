"""Development probe: 2-d exact-order smoother time per level (one 2-sweep call), cfg2 mesh k."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_2508_06049_b200 import klref as K

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sw = int(os.environ.get("GS_SWEEPS", "2"))
levels = [int(x) for x in os.environ.get("GS_LEVELS", "1,2,3,4,5,6,7").split(",")]
h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")), 7)
s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
st = torch.cuda.ExternalStream(s.stream())
tot = 0.0
for l in levels:
    u = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
    b = K.GridFunction(h, l, np.random.rand(h.level_size(l)))
    s.interface_sync(u, K.SYNC_REPLACE)
    s.interface_sync(b, K.SYNC_REPLACE)
    s.gauss_seidel(u, b, 2)
    s.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.gauss_seidel(u, b, sw)
        e1.record(st)
        s.synchronize()
        ts.append(e0.elapsed_time(e1))
    calls = 2 * 2 * (7 - l + 1)  # per FMG (nu=2): (pre + post) x 2 V-cycles x targets >= l
    tot += min(ts) * calls
    print(f"k={k} level {l}: n={2**l} macros={h.num_macros()} GS x{sw} {min(ts)*1e3:8.1f} us  "
          f"(x{calls} calls/FMG = {min(ts)*calls:.2f} ms)", flush=True)
print(f"k={k} smoother total per FMG ~ {tot:.2f} ms")
