"""The C++ drop-in facade (include/klref_b200/klref.hpp) driven through the
reference's own call sequence of run_kl (proj/src/amr.cpp:176-201) by
tests/cpp/dropin_demo: results must equal the patched reference's."""
import json
import os
import subprocess

import numpy as np
import pytest

from _golden import golden, path, rel, sha

DEMO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "dropin_demo")


def _run(args):
    if not os.path.exists(DEMO):
        pytest.skip("tests/cpp/dropin_demo not built (make -C tests/cpp)")
    return subprocess.run([DEMO] + args, capture_output=True, text=True, timeout=300)


def test_dropin_fails_loudly_without_a_device(tmp_path):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    r = _run([path("cfg1.mesh"), "sin", "6", "1", str(tmp_path / "u.bin")])
    assert r.returncode == 1 and "no CUDA device" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,prob,L,nu,key", [("cfg1.mesh", "sin", 6, 1, "cfg1"),
                                                ("cfg2_k3.mesh", "lshape", 7, 2, "cfg2:3")])
def test_dropin_matches_reference(tmp_path, mesh, prob, L, nu, key):
    out = tmp_path / "u.bin"
    r = _run([path(mesh), prob, str(L), str(nu), str(out)])
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    g = golden()
    rec = g["cfg1"] if key == "cfg1" else g["cfg2"][int(key.split(":")[1])]
    u = np.fromfile(out, dtype=np.float64)
    assert sha(u) == rec["sha256"][f"u_{L}"], "u_L differs from the reference"
    nb, nc, th, eta = rec["est_u1"]
    tol = 1e-12 if key == "cfg1" else 1e-9
    assert rel(d["eta"], eta) <= tol and rel(d["norm_base"], nb) <= tol and rel(d["conv"], th) <= tol
    # effectivity_index / make_bounds through the facade (proj/src/estimator.cpp:47-123)
    assert d["gamma"] == d["eta"] / d["exact"] and d["spread"] >= 1.0
    assert round(d["c1"], 2) == 0.53 and round(d["c2"], 2) == 1.67
    ref_loc = np.array(rec["eta_local_u1"])
    assert np.max(np.abs(np.array(d["eta_local"]) - ref_loc) / np.abs(ref_loc)) <= tol
