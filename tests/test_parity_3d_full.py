"""3-d path at the BASELINE sizes: configs 3 (384 macro tets) and 5 (3072), l = 6.

Fixtures: tests/gen_golden_3d.py runs the builder's 3-d C restatement
(oracle/klref_oracle3d.c) once in the build container and stores sha256 of
every level's u and b and of every w snapshot, plus the estimator outputs.
The reference has no 3-d solver (proj/src/hhg.cpp:49-50), so this pins the
device path to the builder's specification, not to the reference.

* faithful f (host-tabulated source): the whole FMG state bit for bit, eta /
  theta / norms to 1e-12 and eta_T elementwise to 1e-10 (the per-macro sums
  are reduced in another order);
* device f (the bench mode): eta and eta_T within 1e-9 (north_star tolerance);
* config 5 sharded as the bench splits it (8 shards, levels <= 3 replicated),
  bit for bit.
"""
import hashlib
import json

import numpy as np
import pytest

from _golden import path
from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients


def fixture(name):
    with open(path(f"{name}_full.json")) as fh:
        return json.load(fh)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def problem(fx):
    if fx["problem"] == "sin3":
        return K.Problem(K.PROBLEM_SIN3D)
    return K.Problem(K.PROBLEM_SERIES3D, series_coefficients(fx["series_seed"]))


def check_estimates(rep, fx, tol_global, tol_local):
    for a, key in ((rep.norm_base, "norm_base"), (rep.norm_coarser, "norm_coarser"), (rep.conv_factor, "theta"),
                   (rep.eta, "eta")):
        assert abs(a - fx[key]) <= tol_global * abs(fx[key]), (key, a, fx[key])
    ref = np.asarray(fx["eta_local"])
    rel = np.max(np.abs(rep.eta_local - ref) / ref)
    assert rel <= tol_local, f"eta_T max rel {rel:.3e}"


def check_state(get_u, get_b, get_w, fx):
    L = fx["level"]
    for l in range(L + 1):
        assert sha(get_b(l)) == fx["sha_b"][l], f"b level {l}"
    for l in range(L):
        assert sha(get_w(l)) == fx["sha_w"][l], f"w snapshot {l}"
    for l in range(L + 1):
        u = get_u(l)
        if l == L and sha(u) != fx["sha_u"][l]:
            head = np.asarray(fx["uL_head"])
            raise AssertionError(f"u level {l}: sha differs; head max diff {np.max(np.abs(u[:16] - head)):.3e}, "
                                 f"max|u| {np.max(np.abs(u)):.17g} vs {fx['uL_max_abs']:.17g}")
        assert sha(u) == fx["sha_u"][l], f"u level {l}"


def test_fixtures_consistent_with_host_hierarchy():
    for name in ("cfg3", "cfg5"):
        fx = fixture(name)
        h = K.GridHierarchy.build(kuhn_cube(fx["cubes"]), fx["level"], device=False)
        assert h.num_macros() == fx["macros"]
        assert h.dof_count(fx["level"]) == fx["dofs"] == (2 ** fx["level"] * fx["cubes"] + 1) ** 3
        assert fx["status"] == 0 and len(fx["eta_local"]) == fx["macros"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_full_size_fmg_bitwise(name):
    fx = fixture(name)
    h = K.GridHierarchy.build(kuhn_cube(fx["cubes"]), fx["level"])
    s = K.MultigridSolver(h, problem(fx), K.SolverConfig(nu=fx["nu"], faithful_source=1))
    st = s.fmg()
    check_state(st.u, st.b, st.w, fx)
    check_estimates(s.error_estimate(1, K.UNSCALED), fx, 1e-12, 1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_full_size_device_source_within_tolerance(name):
    """The bench mode (f from device libm) against the faithful fixture: 1e-9."""
    fx = fixture(name)
    h = K.GridHierarchy.build(kuhn_cube(fx["cubes"]), fx["level"])
    s = K.MultigridSolver(h, problem(fx), K.SolverConfig(nu=fx["nu"], faithful_source=0))
    s.fmg()
    check_estimates(s.error_estimate(1, K.UNSCALED), fx, 1e-9, 1e-9)


@pytest.mark.gpu
def test_cfg5_sharded_as_bench_bitwise():
    """The bench's split of config 5 (8 shards, levels <= 3 replicated, in-process
    transport on one device) reproduces the fixture bit for bit."""
    fx = fixture("cfg5")
    h = K.GridHierarchy.build(kuhn_cube(fx["cubes"]), fx["level"])
    sh = K.ShardedSolver(h, problem(fx), K.SolverConfig(nu=fx["nu"], faithful_source=1), local_shards=8, rep_level=3)
    sh.fmg()
    check_state(lambda l: sh.state(K.STATE_U, l), lambda l: sh.state(K.STATE_B, l),
                lambda l: sh.state(K.STATE_W, l + 1), fx)
    check_estimates(sh.error_estimate(1, K.UNSCALED), fx, 1e-12, 1e-10)
