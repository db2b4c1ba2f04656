"""Generate the config-4 fixtures (tests/golden/cfg4_k*.mesh, cfg4.json).

Test infrastructure (run in the build container, where /root/reference exists):
  bash oracle/build_ref.sh && python tests/gen_golden_cfg4.py

BASELINE.json config 4: unit cube as 6 Kuhn tetrahedra, l = 6, Gaussian peak
u = exp(-1000 |x - c|^2), 4 AMR iterations of (estimate -> mark >= 0.5 max on
the green-reverted set -> refine).  The refinement is the reference's own
refine_rg_3d (proj/src/macro_mesh.cpp:662-676) with its revert_green and
aggregation (proj/src/amr.cpp:41-65), run by oracle/_ref/ref_driver amr3d; the
reference has no 3-d solver, so eta_T comes from the builder's 3-d C oracle
(oracle/klref_oracle3d.c) on each mesh as written and re-read.
"""
import json
import os
import shutil
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLD = os.path.join(HERE, "golden")
DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")
L, NU, K = 6, 2, 4


def parse(path):
    d = {}
    with open(path) as fh:
        for ln in fh:
            p = ln.split()
            if p:
                d[p[0]] = p[1:]
    out = {"num_macros": int(d["num_macros"][0]), "dofs": int(d["dofs"][0]), "eta": float(d["eta"][0]),
           "norm_base": float(d["norm_base"][0]), "norm_coarser": float(d["norm_coarser"][0]),
           "eta_local": [float(x) for x in d["eta_local"]], "active_ids": [int(x) for x in d["active_ids"]],
           "green_parent": [int(x) for x in d["green_parent"]]}
    if "marks_halfmax_eta" in d:
        out["reverted_ids"] = [int(x) for x in d["reverted_ids"]]
        out["marks_halfmax_eta"] = [int(x) for x in d["marks_halfmax_eta"]]
    return out


def main():
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([DRIVER, "amr3d", str(L), str(NU), str(K), tmp], check=True)
        meta = {"level": L, "nu": NU, "problem": "gauss", "steps": []}
        for k in range(K + 1):
            shutil.copy(os.path.join(tmp, f"cfg4_k{k}.mesh"), os.path.join(GOLD, f"cfg4_k{k}.mesh"))
            meta["steps"].append(parse(os.path.join(tmp, f"cfg4_k{k}_report.txt")))
    with open(os.path.join(GOLD, "cfg4.json"), "w") as fh:
        json.dump(meta, fh)


if __name__ == "__main__":
    main()
