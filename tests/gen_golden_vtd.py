"""Generate tests/golden/vtd.json: FinestPolicy::ValidationTwoDigits (the
reference's default finest policy, proj/src/multigrid.cpp:282-293) and the
ExactErrorEvaluator norms after it, from the patched reference
(oracle/_ref/ref_driver solvevtd).  Test infrastructure:
  bash oracle/build_ref.sh && python tests/gen_golden_vtd.py
"""
import hashlib
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLD = os.path.join(HERE, "golden")
DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")
CASES = [("cfg1", "cfg1.mesh", "sin", 6, 1), ("cfg2k0", "cfg2_k0.mesh", "lshape", 7, 2),
         ("cfg2k3", "cfg2_k3.mesh", "lshape", 7, 2)]


def main():
    out = {}
    for name, mesh, prob, L, nu in CASES:
        with tempfile.TemporaryDirectory() as tmp:
            subprocess.run([DRIVER, "solvevtd", os.path.join(GOLD, mesh), prob, str(L), str(nu), tmp], check=True)
            d = {}
            with open(os.path.join(tmp, "report.txt")) as fh:
                for ln in fh:
                    p = ln.split()
                    d[p[0]] = p[1:]
            with open(os.path.join(tmp, f"u_{L}.bin"), "rb") as fh:
                u_sha = hashlib.sha256(fh.read()).hexdigest()
        out[name] = {"mesh": mesh, "problem": prob, "L": L, "nu": nu, "extra_cycles": int(d["extra_cycles"][0]),
                     "exact_global": float(d["exact_global"][0]),
                     "exact_local": [float(x) for x in d["exact_local"]], "u_sha256": u_sha}
    with open(os.path.join(GOLD, "vtd.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
