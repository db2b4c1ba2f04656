"""Development probe: one GS sweep on a cfg2 level, pipelined kernel vs the macro-DAG fallback; first differences."""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np

from paper_2508_06049_b200 import klref as K

k, l, sweeps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
if os.environ.get("CHILD"):
    mesh = os.environ.get("MESH") or os.path.join(REPO, "tests", "golden", f"cfg2_k{k}.mesh")
    h = K.GridHierarchy.build(K.MacroMesh.read(mesh), 7)
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_LSHAPE), K.SolverConfig(nu=2))
    rng = np.random.default_rng(1)
    u = K.GridFunction(h, l, rng.random(h.level_size(l)))
    b = K.GridFunction(h, l, rng.random(h.level_size(l)))
    s.interface_sync(u, K.SYNC_REPLACE)
    s.interface_sync(b, K.SYNC_REPLACE)
    s.gauss_seidel(u, b, sweeps)
    np.save(os.environ["CHILD"], u.numpy())
    sys.exit(0)
outs = []
for pipe in ("1", "0"):
    f = f"/tmp/gsdiff_{pipe}.npy"
    env = dict(os.environ, CHILD=f, KB_GS_PIPE=pipe, KB_GS_SCHED="0")
    subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, check=True)
    outs.append(np.load(f))
a, b = outs
n = 2 ** l
S = (n + 1) * (n + 2) // 2
d = np.nonzero(a != b)[0]
print(f"differences: {d.size} of {a.size}")
M = a.size // S
lat = np.zeros(S, dtype=bool)
q = 0
for j in range(n + 1):
    for i in range(n + 1 - j):
        lat[q] = i >= 1 and j >= 1 and i + j <= n - 1
        q += 1
bad = (a != b).reshape(M, S)
per = [(m, int(bad[m][lat].sum()), int(bad[m][~lat].sum())) for m in range(M)]
print("first macros with interior differences:", [x for x in per if x[1] > 0][:8])
print("macros with boundary-only differences:", [x for x in per if x[1] == 0 and x[2] > 0][:12])
for q in d[:40]:
    m, idx = divmod(int(q), S)
    j = 0
    while idx >= n + 1 - j:
        idx -= n + 1 - j
        j += 1
    print(f"macro {m} (i={idx}, j={j}) t={idx + 2 * j}: pipe {a[q]!r} dag {b[q]!r}")
