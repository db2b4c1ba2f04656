"""ExactErrorEvaluator (proj/src/fem.cpp:358-476) and FinestPolicy::
ValidationTwoDigits (proj/src/multigrid.cpp:282-293, the reference's default
finest policy) on the device, against the patched reference (tests/golden:
golden.json exact norms after FMG with policy None; vtd.json from
oracle/_ref/ref_driver solvevtd).

The three-term moment form cancels: the device keeps
the reference's sequential per-macro sums, so the norms must agree to
rounding of the host-side global sum only.
"""
import json

import numpy as np
import pytest

from _golden import golden, path, sha
from paper_2508_06049_b200 import klref as K

TOL = 1e-12


def _solve(mesh, L, prob, nu, policy):
    h = K.GridHierarchy.build(K.MacroMesh.read(path(mesh)), L)
    s = K.MultigridSolver(h, K.Problem(prob), K.SolverConfig(nu=nu, faithful_source=1, finest_policy=policy))
    s.fmg()
    return h, s


def _rel(a, b):
    return abs(a - b) / abs(b)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [None, 0, 3, 5])
def test_exact_error_after_fmg(k):
    g = golden()
    if k is None:
        ref, mesh, prob, L, nu = g["cfg1"], "cfg1.mesh", K.PROBLEM_SIN2D, 6, 1
    else:
        ref, mesh, prob, L, nu = g["cfg2"][k], f"cfg2_k{k}.mesh", K.PROBLEM_LSHAPE, 7, 2
    _, s = _solve(mesh, L, prob, nu, K.POLICY_NONE)
    glob, loc = s.exact_error()
    ref_g = ref["exact_global"][0] if isinstance(ref["exact_global"], list) else ref["exact_global"]
    assert _rel(glob, ref_g) <= TOL
    ref_l = np.asarray(ref["exact_local"])
    assert np.max(np.abs(loc - ref_l) / ref_l) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "cfg2k0", "cfg2k3"])
def test_validation_two_digits_policy(name):
    with open(path("vtd.json")) as fh:
        ref = json.load(fh)[name]
    prob = {"sin": K.PROBLEM_SIN2D, "lshape": K.PROBLEM_LSHAPE}[ref["problem"]]
    h, s = _solve(ref["mesh"], ref["L"], prob, ref["nu"], K.POLICY_VALIDATION_TWO_DIGITS)
    assert s.extra_cycles() == ref["extra_cycles"]
    assert sha(s.state(K.STATE_U, ref["L"])) == ref["u_sha256"], "u_L after the extra cycles"
    glob, loc = s.exact_error()
    assert _rel(glob, ref["exact_global"]) <= TOL
    assert np.max(np.abs(loc - np.asarray(ref["exact_local"])) / np.asarray(ref["exact_local"])) <= TOL


def test_policy_config_plumbing():
    """The config struct carries the policy and max_extra_cycles (ABI layout)."""
    c = K.SolverConfig(finest_policy=K.POLICY_VALIDATION_TWO_DIGITS, max_extra_cycles=7).c()
    assert c.finest_policy == 1 and c.max_extra_cycles == 7


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rve_cfg1", "rve_cfg2k3"])
def test_residual_vs_estimate_policy(name):
    """FinestPolicy::ResidualVsEstimate (proj/src/multigrid.cpp:294-319): the same
    number of extra finest V-cycles and the same u_L (sha256) as the patched
    reference (oracle/_ref/ref_driver solverve)."""
    with open(path("vtd.json")) as fh:
        ref = json.load(fh)[name]
    prob = {"sin": K.PROBLEM_SIN2D, "lshape": K.PROBLEM_LSHAPE}[ref["problem"]]
    h, s = _solve(ref["mesh"], ref["L"], prob, ref["nu"], K.POLICY_RESIDUAL_VS_ESTIMATE)
    assert s.extra_cycles() == ref["extra_cycles"]
    assert sha(s.state(K.STATE_U, ref["L"])) == ref["u_sha256"], "u_L after the extra cycles"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rve_cfg1", "rve_cfg2k3"])
def test_solve_direct(name):
    """MultigridSolver::solve_direct (proj/src/multigrid.cpp:323-357): level 0 by
    the coarse CG, bit for bit; level l > 0 by the reference's level CG, within
    1e-12 (its dot products are reduced in another order on the device)."""
    with open(path("vtd.json")) as fh:
        ref = json.load(fh)[name]
    prob = {"sin": K.PROBLEM_SIN2D, "lshape": K.PROBLEM_LSHAPE}[ref["problem"]]
    h = K.GridHierarchy.build(K.MacroMesh.read(path(ref["mesh"])), ref["L"])
    s = K.MultigridSolver(h, K.Problem(prob), K.SolverConfig(nu=ref["nu"], faithful_source=1))
    u0 = s.solve_direct(0).numpy()
    assert np.array_equal(u0, np.asarray(ref["direct_0"]))
    ul = s.solve_direct(ref["l_direct"]).numpy()
    assert np.max(np.abs(ul[:32] - np.asarray(ref["direct_l_head"]))) <= 1e-12 * ref["direct_l_max_abs"]
    assert abs(np.max(np.abs(ul)) - ref["direct_l_max_abs"]) <= 1e-12 * ref["direct_l_max_abs"]
