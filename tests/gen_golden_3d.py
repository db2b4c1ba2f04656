"""Generate the full-size 3-d fixtures (tests/golden/cfg3_full.json, cfg5_full.json).

Test infrastructure (run in the build container; takes minutes, single thread):
  make -C oracle && python tests/gen_golden_3d.py [cfg3|cfg5]

BASELINE.json config 3: unit cube as 4^3 Kuhn cubes (384 macro tets), l = 6,
u = sin(pi x) sin(pi y) sin(pi z).  Config 5: 8^3 Kuhn cubes (3072 macro tets),
l = 6, f = seeded 4x4x4 sine series (meshes.series_coefficients()), g = 0.
The reference has no 3-d solver (proj/src/hhg.cpp:49-50), so the values come
from the builder's 3-d C restatement (oracle/klref_oracle3d.c, faithful f,
FinestPolicy::None, nu = 2, V(2,2)) -- the same specification the device path
follows; the fixture pins the device path at the BASELINE size bit for bit
(sha256 of u, b of every level and of every w snapshot) plus the estimator
(eta, theta, eta_T) of proj/src/estimator.cpp:8-45's algebra.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

from oracle import oracle as O  # noqa: E402
from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients  # noqa: E402

CONFIGS = {
    "cfg3": {"cubes": 4, "level": 6, "problem": "sin3", "params": None},
    "cfg5": {"cubes": 8, "level": 6, "problem": "series", "params": "default_seed"},
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def generate(name):
    c = CONFIGS[name]
    mesh = kuhn_cube(c["cubes"])
    L = c["level"]
    par = series_coefficients() if c["params"] else None
    t0 = time.time()
    o = O.Hier3D(mesh.coords, mesh.elements, L)
    t1 = time.time()
    st = O.fmg3d(o, c["problem"], params=par, nu=2)
    t2 = time.time()
    e = O.estimate3d(st)
    t3 = time.time()
    uL = st["u"][L]
    out = {
        "config": name, "cubes": c["cubes"], "macros": int(mesh.elements.shape[0]), "level": L, "nu": 2,
        "problem": c["problem"], "series_seed": 20240817 if par is not None else None,
        "dofs": int(o.dofs(L)), "status": int(st["status"]),
        "sha_u": [sha(st["u"][l]) for l in range(L + 1)],
        "sha_b": [sha(st["b"][l]) for l in range(L + 1)],
        "sha_w": [sha(st["w"][l]) for l in range(L)],
        "uL_max_abs": float(np.max(np.abs(uL))), "uL_sum": float(np.sum(uL)),
        "uL_head": [float(x) for x in uL[:16]],
        "norm_base": e["norm_base"], "norm_coarser": e["norm_coarser"], "theta": e["conv"], "eta": e["eta"],
        "eta_local": [float(x) for x in e["local_base"]],
        "oracle_seconds": {"build": t1 - t0, "fmg": t2 - t1, "estimate": t3 - t2},
    }
    with open(os.path.join(HERE, "golden", f"{name}_full.json"), "w") as fh:
        json.dump(out, fh)
    print(f"{name}: dofs {out['dofs']} eta {out['eta']:.12e} theta {out['theta']:.10f} "
          f"(build {t1 - t0:.0f}s, fmg {t2 - t1:.0f}s, estimate {t3 - t2:.0f}s)", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CONFIGS):
        generate(nm)
