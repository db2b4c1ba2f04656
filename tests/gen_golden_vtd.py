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
    # FinestPolicy::ResidualVsEstimate (proj/src/multigrid.cpp:294-319) and
    # solve_direct(0), solve_direct(l) (proj/src/multigrid.cpp:323-357)
    for name, mesh, prob, L, nu, ld in [("cfg1", "cfg1.mesh", "sin", 6, 1, 3),
                                        ("cfg2k3", "cfg2_k3.mesh", "lshape", 7, 2, 2)]:
        with tempfile.TemporaryDirectory() as tmp:
            subprocess.run([DRIVER, "solverve", os.path.join(GOLD, mesh), prob, str(L), str(nu), str(ld), tmp],
                           check=True)
            with open(os.path.join(tmp, "report.txt")) as fh:
                d = {ln.split()[0]: ln.split()[1:] for ln in fh if ln.strip()}

            def h(f):
                with open(os.path.join(tmp, f), "rb") as fh:
                    return hashlib.sha256(fh.read()).hexdigest()

            def arr(f):
                import numpy as np
                return [float(x) for x in np.fromfile(os.path.join(tmp, f), dtype=np.float64)]

            out["rve_" + name] = {"mesh": mesh, "problem": prob, "L": L, "nu": nu, "l_direct": ld,
                                  "extra_cycles": int(d["extra_cycles"][0]), "u_sha256": h(f"u_{L}.bin"),
                                  "direct_0": arr("direct_0.bin"), "direct_l_sha256": h(f"direct_{ld}.bin"),
                                  "direct_l_max_abs": max(abs(x) for x in arr(f"direct_{ld}.bin")),
                                  "direct_l_head": arr(f"direct_{ld}.bin")[:32]}
    with open(os.path.join(GOLD, "vtd.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
