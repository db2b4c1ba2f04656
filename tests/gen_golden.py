"""Generate the golden fixtures under tests/golden/ from the patched reference.

Test infrastructure (run in the build container, where /root/reference exists):
  bash oracle/build_ref.sh && python tests/gen_golden.py

It runs oracle/_ref/ref_driver (the reference's own sources + the D1/D2
one-line fixes) through the reference's public API and stores:
  - the config meshes (reference mesh_io format) incl. the cfg2 AMR sequence;
  - per solve: scalars of every error_estimate(j, kind), eta_local, exact
    errors, marks, genealogy needed for marking, and sha256 of every u/b/w
    level array (bitwise pins);
  - small full arrays (npz) for the seeded single-operation tests
    (apply/residual/GS/restrict/prolong/cg0/dot) at reduced levels, and
    hashes of the same operations at the full config levels.
"""
import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLD = os.path.join(HERE, "golden")
DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")
DRIVER_FMA = os.path.join(REPO, "oracle", "_ref", "ref_driver_fma")


def run(*args, driver=DRIVER):
    subprocess.run([driver, *map(str, args)], check=True)


def sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def parse_report(path):
    out = {}
    with open(path) as fh:
        for ln in fh:
            parts = ln.split()
            if not parts:
                continue
            key, vals = parts[0], parts[1:]
            if key.startswith(("marks_", "active_", "reverted_")):
                out[key] = [int(v) for v in vals]
            elif key in ("num_macros", "dofs"):
                out[key] = int(vals[0])
            else:
                out[key] = [float(v) for v in vals]
    return out


def solve_record(d, L, report=None):
    rec = parse_report(report or os.path.join(d, "report.txt"))
    rec["sha256"] = {}
    for l in range(L + 1):
        for c in ("u", "b") + (("w",) if l < L else ()):
            rec["sha256"][f"{c}_{l}"] = sha(os.path.join(d, f"{c}_{l}.bin"))
    return rec


def ops_fixture(tmp, mesh, L, seed, small_L, name):
    d = os.path.join(tmp, "ops_" + name)
    run("ops", mesh, L, seed, d)
    arrays, hashes = {}, {}
    for f in sorted(os.listdir(d)):
        p = os.path.join(d, f)
        stem = f.rsplit(".", 1)[0]
        if f.endswith(".txt"):
            arrays[stem] = np.array([float(open(p).read())])
            continue
        lvl = int(stem.split("_")[-1]) if "_" in stem else 0
        hashes[stem] = sha(p)
        if lvl <= small_L:
            arrays[stem] = np.fromfile(p, dtype=np.float64)
    np.savez_compressed(os.path.join(GOLD, f"ops_{name}.npz"), **arrays)
    return {"seed": seed, "L": L, "small_L": small_L, "sha256": hashes}


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build oracle/_ref first: bash oracle/build_ref.sh")
    os.makedirs(GOLD, exist_ok=True)
    tmp = tempfile.mkdtemp(prefix="klref_golden_")
    try:
        gold = {"generator": "tests/gen_golden.py via oracle/_ref/ref_driver (reference + D1/D2)"}
        # config 1: 8 triangles, L = 6, nu = 1, sin problem
        run("mesh", "cfg1", os.path.join(GOLD, "cfg1.mesh"))
        d = os.path.join(tmp, "cfg1")
        run("solve", os.path.join(GOLD, "cfg1.mesh"), "sin", 6, 1, d)
        gold["cfg1"] = solve_record(d, 6)
        shutil.copy(os.path.join(d, "refined_top10_eta.mesh"), os.path.join(GOLD, "cfg1_refined.mesh"))
        np.savez_compressed(os.path.join(GOLD, "cfg1_state.npz"),
                            u_6=np.fromfile(os.path.join(d, "u_6.bin")),
                            w_5=np.fromfile(os.path.join(d, "w_5.bin")),
                            w_4=np.fromfile(os.path.join(d, "w_4.bin")),
                            b_6=np.fromfile(os.path.join(d, "b_6.bin")))
        # FMA-contracted reference build: the reference's own rounding noise floor
        dfma = os.path.join(tmp, "cfg1_fma")
        run("solve", os.path.join(GOLD, "cfg1.mesh"), "sin", 6, 1, dfma, driver=DRIVER_FMA)
        gold["cfg1_fma"] = parse_report(os.path.join(dfma, "report.txt"))

        # config 2: L-shape, 6 triangles, L = 7, nu = 2, 5 AMR steps, >= 0.5 max marking
        run("mesh", "cfg2", os.path.join(tmp, "cfg2.mesh"))
        d2 = os.path.join(tmp, "cfg2")
        run("amr", os.path.join(tmp, "cfg2.mesh"), "lshape", 7, 2, 5, "halfmax", d2)
        d2f = os.path.join(tmp, "cfg2_fma")
        run("amr", os.path.join(tmp, "cfg2.mesh"), "lshape", 7, 2, 5, "halfmax", d2f, driver=DRIVER_FMA)
        gold["cfg2"] = []
        for k in range(6):
            shutil.copy(os.path.join(d2, f"k{k}_mesh.txt"), os.path.join(GOLD, f"cfg2_k{k}.mesh"))
            rec = solve_record(os.path.join(d2, f"k{k}"), 7, os.path.join(d2, f"k{k}_report.txt"))
            rec["fma"] = {kk: v for kk, v in parse_report(os.path.join(d2f, f"k{k}_report.txt")).items()
                          if kk.startswith("est_") or kk.startswith("eta_local_u1")}
            gold["cfg2"].append(rec)
        np.savez_compressed(os.path.join(GOLD, "cfg2_k0_state.npz"),
                            u_7=np.fromfile(os.path.join(d2, "k0", "u_7.bin")))

        # seeded single operations (random x, replace-synced)
        gold["ops_cfg1"] = ops_fixture(tmp, os.path.join(GOLD, "cfg1.mesh"), 6, 12345, 4, "cfg1")
        gold["ops_cfg2k3"] = ops_fixture(tmp, os.path.join(GOLD, "cfg2_k3.mesh"), 7, 777, 4, "cfg2k3")
        with open(os.path.join(GOLD, "golden.json"), "w") as fh:
            json.dump(gold, fh, indent=1, sort_keys=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print("wrote", GOLD)


if __name__ == "__main__":
    main()
