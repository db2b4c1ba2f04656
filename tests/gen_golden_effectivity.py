"""Generate tests/golden/effectivity.json: effectivity_constants, the local
spread bounds, make_bounds' order (proj/src/estimator.cpp:47-99) and
effectivity_index (:100-123) computed by the reference itself
(oracle/_ref/ref_driver bounds / effidx).  Test infrastructure:
  bash oracle/build_ref.sh && python tests/gen_golden_effectivity.py
"""
import json
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")


def main():
    triples = []
    for theta in (0.25, 2.0 ** (-4.0 / 3.0), 0.1, 0.5, 0.9):
        for eps in (0.0, 0.05, 0.3):
            for j in (1, 2, 3, 4):
                triples.append((theta, eps, j))
    triples += [(0.0, 0.0, 1), (0.25, -0.1, 1), (0.25, 0.0, 0), (0.8, 0.3, 1), (1.0, 0.0, 2)]  # DomainError
    inp = "".join(f"{t!r} {e!r} {j}\n" for t, e, j in triples)
    out = subprocess.run([DRIVER, "bounds"], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    bounds = []
    for (t, e, j), ln in zip(triples, out):
        p = ln.split()
        bounds.append({"theta": t, "eps": e, "offset": j, "error": p[0] == "ERR",
                       "values": None if p[0] == "ERR" else [float(x) for x in p[:4]] + [int(p[4])]})
    rng = np.random.default_rng(11)
    cases = []
    for n, m, zero_global in ((8, 8, False), (6, 4, False), (5, 5, True), (12, 12, False)):
        eta_local = rng.uniform(0.0, 1.0, n)
        per = rng.uniform(0.0, 1.0, m)
        per[0] = 0.0                  # excluded: exactly zero
        if m > 2:
            per[2] = 1e-20            # excluded: below 1e-14 of the global error
        glob = 0.0 if zero_global else float(np.sqrt(np.sum(per ** 2)))
        eta = float(np.sqrt(np.sum(eta_local ** 2)))
        with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as fh:
            fh.write(f"{eta!r} {n} " + " ".join(repr(float(v)) for v in eta_local) +
                     f" {glob!r} {m} " + " ".join(repr(float(v)) for v in per) + "\n")
            path = fh.name
        p = subprocess.run([DRIVER, "effidx", path], capture_output=True, text=True, check=True).stdout.split()
        os.unlink(path)
        cases.append({"eta": eta, "eta_local": eta_local.tolist(), "exact_global": glob, "exact_local": per.tolist(),
                      "gamma": float(p[0]), "gamma_valid": p[1] == "1", "spread": float(p[2]),
                      "spread_valid": p[3] == "1", "gamma_local": [float(x) for x in p[4:]]})
    with open(os.path.join(HERE, "golden", "effectivity.json"), "w") as fh:
        json.dump({"source": "patched reference, oracle/_ref/ref_driver bounds|effidx", "bounds": bounds,
                   "effectivity_index": cases}, fh, indent=1)


if __name__ == "__main__":
    main()
