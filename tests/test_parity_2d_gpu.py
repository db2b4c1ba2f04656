"""GPU parity of the 2-d hot path against the patched reference (goldens from oracle/_ref).

Bitwise targets: apply, residual, Gauss-Seidel,
restriction, prolongation, level-0 CG, and the whole FMG state (u, b, w of every
level) are compared byte for byte (sha256 / array_equal) with the reference.
Reductions that the device does in a different order (dot_unique over the
whole level, the estimator norms) are checked to a relative 1e-12 / 1e-9
(north_star tolerances: apply <= 1e-12, FMG and estimates <= 1e-9).
Marks must be identical sets.
"""
import numpy as np
import pytest

from _golden import golden, npz, path, rel, rel_max, sha
from _rng import splitmix_uniform
from paper_2508_06049_b200 import klref as K

pytestmark = pytest.mark.gpu

TOL_APPLY = 1e-12
TOL_FMG = 1e-9


def _hier(mesh_file, L):
    return K.GridHierarchy.build(K.MacroMesh.read(path(mesh_file)), L)


def _solver(h, problem=K.PROBLEM_ZERO, **cfg):
    return K.MultigridSolver(h, K.Problem(problem), K.SolverConfig(**cfg))


OPS = [("cfg1", "cfg1.mesh"), ("cfg2k3", "cfg2_k3.mesh")]


@pytest.mark.parametrize("name,mesh", OPS)
def test_single_operations_small_levels_bitwise(name, mesh):
    """Every single operation at levels 0..4 equals the reference byte for byte."""
    g = golden()["ops_" + name]
    data = npz(f"ops_{name}.npz")
    h = _hier(mesh, g["L"])
    s = _solver(h)
    for l in range(g["small_L"] + 1):
        x = K.GridFunction(h, l, data[f"x_{l}"])
        bb = K.GridFunction(h, l, data[f"bb_{l}"])
        y = h.create_function(l)
        s.apply(K.STIFFNESS, x, y)
        assert np.array_equal(y.numpy(), data[f"Ax_{l}"]), f"stiffness apply level {l}"
        s.apply(K.MASS, x, y)
        assert np.array_equal(y.numpy(), data[f"Mx_{l}"]), f"mass apply level {l}"
        s.residual(x, bb, y)
        assert np.array_equal(y.numpy(), data[f"res_{l}"]), f"residual level {l}"
        d = s.dot_unique(x, bb)
        assert rel(d, float(data[f"dot_{l}"][0])) <= TOL_APPLY
        if l >= 1:
            u = K.GridFunction(h, l, data[f"x_{l}"])
            s.gauss_seidel(u, bb, 1)
            assert np.array_equal(u.numpy(), data[f"gs1_{l}"]), f"GS sweep 1 level {l}"
            s.gauss_seidel(u, bb, 1)
            assert np.array_equal(u.numpy(), data[f"gs2_{l}"]), f"GS sweep 2 level {l}"
            u2 = K.GridFunction(h, l, data[f"x_{l}"])
            s.gauss_seidel(u2, bb, 2)
            assert np.array_equal(u2.numpy(), data[f"gs2_{l}"]), f"GS 2 sweeps in one launch, level {l}"
            rc = h.create_function(l - 1)
            s.restrict_transpose(x, rc)
            assert np.array_equal(rc.numpy(), data[f"restrict_{l}"]), f"restriction {l}->{l-1}"
        if l < g["L"]:
            f = h.create_function(l + 1)
            s.prolongate(x, f)
            assert np.array_equal(f.numpy(), data[f"prolong_{l}"]), f"prolongation {l}->{l+1}"
        if l == 0:
            u0 = h.create_function(0)
            s.cg_level0(u0, bb)
            assert np.array_equal(u0.numpy(), data["cg0"]), "level-0 CG"


@pytest.mark.parametrize("name,mesh", OPS)
def test_single_operations_full_levels_bitwise(name, mesh):
    """Seeded random inputs at every level up to the config's L, compared by sha256."""
    g = golden()["ops_" + name]
    hashes = g["sha256"]
    h = _hier(mesh, g["L"])
    s = _solver(h)
    start = 0
    for l in range(g["L"] + 1):
        N = h.level_size(l)
        xs = splitmix_uniform(g["seed"], start, N)
        bs = splitmix_uniform(g["seed"], start + N, N)
        start += 2 * N
        if l <= g["small_L"]:
            continue
        x = K.GridFunction(h, l, xs)
        bb = K.GridFunction(h, l, bs)
        s.interface_sync(x, K.SYNC_REPLACE)
        s.interface_sync(bb, K.SYNC_REPLACE)
        assert sha(x.numpy()) == hashes[f"x_{l}"], f"replace sync level {l}"
        assert sha(bb.numpy()) == hashes[f"bb_{l}"]
        y = h.create_function(l)
        s.apply(K.STIFFNESS, x, y)
        assert sha(y.numpy()) == hashes[f"Ax_{l}"], f"stiffness apply level {l}"
        s.apply(K.MASS, x, y)
        assert sha(y.numpy()) == hashes[f"Mx_{l}"], f"mass apply level {l}"
        s.residual(x, bb, y)
        assert sha(y.numpy()) == hashes[f"res_{l}"], f"residual level {l}"
        u = K.GridFunction(h, l, x.numpy())
        s.gauss_seidel(u, bb, 1)
        assert sha(u.numpy()) == hashes[f"gs1_{l}"], f"GS level {l}"
        s.gauss_seidel(u, bb, 1)
        assert sha(u.numpy()) == hashes[f"gs2_{l}"], f"GS level {l}"
        rc = h.create_function(l - 1)
        s.restrict_transpose(x, rc)
        assert sha(rc.numpy()) == hashes[f"restrict_{l}"], f"restriction level {l}"
        if l < g["L"]:
            f = h.create_function(l + 1)
            s.prolongate(x, f)
            assert sha(f.numpy()) == hashes[f"prolong_{l}"], f"prolongation level {l}"


def _check_estimates(s, rec, L, tol):
    for j in range(1, L):
        for kind, tag in ((K.UNSCALED, "u"), (K.SCALED, "s")):
            rep = s.error_estimate(j, kind)
            nb, nc, th, eta = rec[f"est_{tag}{j}"]
            assert rel(rep.norm_base, nb) <= tol
            assert rel(rep.norm_coarser, nc) <= tol
            assert rel(rep.conv_factor, th) <= tol
            assert rel(rep.eta, eta) <= tol
            ref_loc = np.array(rec[f"eta_local_{tag}{j}"])
            assert np.max(np.abs(rep.eta_local - ref_loc) / np.abs(ref_loc)) <= tol


def test_fmg_config1_bitwise_faithful():
    """Config 1: FMG state bitwise equal to the reference (host-tabulated f)."""
    rec = golden()["cfg1"]
    h = _hier("cfg1.mesh", 6)
    s = _solver(h, K.PROBLEM_SIN2D, nu=1, faithful_source=1)
    st = s.fmg()
    for l in range(7):
        assert sha(st.u(l)) == rec["sha256"][f"u_{l}"], f"u level {l}"
        assert sha(st.b(l)) == rec["sha256"][f"b_{l}"], f"b level {l}"
        if l < 6:
            assert sha(st.w(l)) == rec["sha256"][f"w_{l}"], f"w level {l}"
    _check_estimates(s, rec, 6, 1e-12)


def test_fmg_config1_device_source():
    """Config 1 with f evaluated on the device (CUDA libm): u_L and estimates within 1e-9."""
    rec = golden()["cfg1"]
    h = _hier("cfg1.mesh", 6)
    s = _solver(h, K.PROBLEM_SIN2D, nu=1, faithful_source=0)
    st = s.fmg()
    assert rel_max(st.u(6), npz("cfg1_state.npz")["u_6"]) <= TOL_FMG
    _check_estimates(s, rec, 6, TOL_FMG)


def test_fmg_config1_marks():
    rec = golden()["cfg1"]
    h = _hier("cfg1.mesh", 6)
    s = _solver(h, K.PROBLEM_SIN2D, nu=1, faithful_source=1)
    s.fmg()
    rep = s.error_estimate(1, K.UNSCALED)
    marks = K.mark(K.MARK_TOP_FRACTION, 0.10, rec["active_ids"], rec["active_green_parent"], rep.eta_local,
                   rec["reverted_ids"])
    assert marks == rec["marks_top10_eta"] == [3]


@pytest.mark.parametrize("k", range(6))
def test_fmg_config2_amr_steps(k):
    """Config 2 (L-shape, L=7, nu=2): every AMR step's FMG state bitwise, estimates
    within 1e-9 and the >= 0.5 max marked set identical."""
    rec = golden()["cfg2"][k]
    h = _hier(f"cfg2_k{k}.mesh", 7)
    assert h.dof_count(7) == rec["dofs"]
    s = _solver(h, K.PROBLEM_LSHAPE, nu=2)
    st = s.fmg()
    for l in range(8):
        assert sha(st.u(l)) == rec["sha256"][f"u_{l}"], f"u level {l}"
        if l < 7:
            assert sha(st.w(l)) == rec["sha256"][f"w_{l}"], f"w level {l}"
    assert sha(st.b(7)) == rec["sha256"]["b_7"]
    _check_estimates(s, rec, 7, TOL_FMG)
    rep = s.error_estimate(1, K.UNSCALED)
    marks = K.mark(K.MARK_HALF_MAX, 0.0, rec["active_ids"], rec["active_green_parent"], rep.eta_local,
                   rec["reverted_ids"])
    assert marks == rec["marks_halfmax_eta"]


def test_fmg_repeatable_and_graph_equals_stream():
    """Graph replay and direct stream launch give identical bits, run after run."""
    h = _hier("cfg2_k2.mesh", 6)
    a = _solver(h, K.PROBLEM_LSHAPE, nu=2, use_graph=1)
    b = _solver(h, K.PROBLEM_LSHAPE, nu=2, use_graph=0)
    ua = a.fmg().u(6)
    ua2 = a.fmg().u(6)
    ub = b.fmg().u(6)
    assert np.array_equal(ua, ua2) and np.array_equal(ua, ub)
