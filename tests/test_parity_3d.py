"""3-d path (BASELINE.json configs 3-5): GPU kernels vs the 3-d CPU oracle.

The reference has no 3-d solver (proj/src/hhg.cpp:49-50), so these tests pin
the device path to the builder's own CPU restatement (oracle/klref_oracle3d.c;
parity unpinned against the reference).  Integer/structure work and
every floating-point operation order are shared specification: single
operations and the whole FMG state must agree bit for bit; reductions done in a
different order (estimator norms, dot products) within 1e-12.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients


def _perturbed_kuhn(N=2, eps=0.03, seed=3):
    """Kuhn mesh with interior vertices moved: not on a grid -> greedy colouring."""
    m = kuhn_cube(N)
    xyz = m.coords.copy()
    rng = np.random.default_rng(seed)
    inner = np.all((xyz > 1e-12) & (xyz < 1 - 1e-12), axis=1)
    xyz[inner] += eps * rng.uniform(-1, 1, size=(inner.sum(), 3))
    return K.MacroMesh(xyz, m.elements.copy(), 3)


MESHES = {"kuhn2": lambda: kuhn_cube(2), "perturbed": _perturbed_kuhn}


def _smooth(X, seed):
    a = np.random.default_rng(seed).normal(size=(3, 3))
    return np.sin(X @ a[0]) + np.cos(X @ a[1]) * X[:, 2] + 0.1 * X[:, 0]


# ---------------------------------------------------------------- CPU (no device)
@pytest.mark.parametrize("name", list(MESHES))
def test_host_hierarchy_matches_oracle(name):
    mesh = MESHES[name]()
    h = K.GridHierarchy.build(mesh, 3, device=False)
    o = O.Hier3D(mesh.coords, mesh.elements, 3)
    for l in range(4):
        assert h.dof_count(l) == o.dofs(l)
        assert h.level_size(l) == o.size(l)
    ptr, mem = h.groups(3)
    assert len(ptr) - 1 > 0 and mem.shape[1] == 4


def test_oracle_3d_invariants():
    """Symmetry, A 1 = 0, 1^T M 1 = |Omega|, P/R adjointness, O(h^2) FMG error."""
    m = kuhn_cube(2)
    o = O.Hier3D(m.coords, m.elements, 3)
    X = o.coords(3)
    x, y = _smooth(X, 1), _smooth(X, 2)
    assert abs(o.dot(3, x, o.apply(3, y)) - o.dot(3, y, o.apply(3, x))) < 1e-12
    assert np.max(np.abs(o.apply(3, np.ones(o.size(3))))) < 1e-13
    assert abs(o.dot(3, np.ones(o.size(3)), o.apply(3, np.ones(o.size(3)), mass=True)) - 1.0) < 1e-13
    c = _smooth(o.coords(2), 3)
    assert abs(o.dot(2, o.restrict(3, x), c) - o.dot(3, x, o.prolongate(2, c))) < 1e-11
    errs = []
    for L in (2, 3, 4):
        oh = O.Hier3D(m.coords, m.elements, L)
        st = O.fmg3d(oh, "sin3", nu=2)
        Y = oh.coords(L)
        errs.append(np.max(np.abs(st["u"][L] - np.prod(np.sin(np.pi * Y), axis=1))))
    assert errs[1] < errs[0] / 3 and errs[2] < errs[1] / 3


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", list(MESHES))
def test_single_operations_bitwise(name):
    mesh = MESHES[name]()
    L = 3
    o = O.Hier3D(mesh.coords, mesh.elements, L)
    h = K.GridHierarchy.build(mesh, L)
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_ZERO), K.SolverConfig(nu=2))
    for l in range(L + 1):
        X = o.coords(l)
        x, bb = _smooth(X, 10 + l), _smooth(X, 20 + l)
        gx, gb, gy = K.GridFunction(h, l, x), K.GridFunction(h, l, bb), h.create_function(l)
        s.apply(K.STIFFNESS, gx, gy)
        assert np.array_equal(gy.numpy(), o.apply(l, x)), f"stiffness apply level {l}"
        s.apply(K.MASS, gx, gy)
        assert np.array_equal(gy.numpy(), o.apply(l, x, mass=True)), f"mass apply level {l}"
        s.residual(gx, gb, gy)
        assert np.array_equal(gy.numpy(), o.residual(l, x, bb)), f"residual level {l}"
        assert abs(s.dot_unique(gx, gb) - o.dot(l, x, bb)) <= 1e-12 * max(1.0, abs(o.dot(l, x, bb)))
        if l >= 1:
            gu = K.GridFunction(h, l, x)
            s.gauss_seidel(gu, gb, 1)
            ref1 = o.gauss_seidel(l, x, bb, 1)
            assert np.array_equal(gu.numpy(), ref1), f"GS sweep level {l}"
            s.gauss_seidel(gu, gb, 1)
            assert np.array_equal(gu.numpy(), o.gauss_seidel(l, ref1, bb, 1)), f"GS second sweep level {l}"
            gc = h.create_function(l - 1)
            s.restrict_transpose(gx, gc)
            assert np.array_equal(gc.numpy(), o.restrict(l, x)), f"restriction {l}->{l - 1}"
        if l < L:
            gf = h.create_function(l + 1)
            s.prolongate(gx, gf)
            assert np.array_equal(gf.numpy(), o.prolongate(l, x)), f"prolongation {l}->{l + 1}"


@pytest.mark.gpu
@pytest.mark.parametrize("name,prob,params", [("kuhn2", "sin3", None), ("perturbed", "gauss", None),
                                              ("kuhn2", "series", "seed")])
def test_fmg_state_bitwise_and_estimates(name, prob, params):
    mesh = MESHES[name]()
    L = 4
    par = series_coefficients(7) if params == "seed" else None
    kind = {"sin3": K.PROBLEM_SIN3D, "gauss": K.PROBLEM_GAUSS3D, "series": K.PROBLEM_SERIES3D}[prob]
    h = K.GridHierarchy.build(mesh, L)
    s = K.MultigridSolver(h, K.Problem(kind, par), K.SolverConfig(nu=2, faithful_source=1))
    st = s.fmg()
    o = O.Hier3D(mesh.coords, mesh.elements, L)
    ref = O.fmg3d(o, prob, params=par, nu=2)
    for l in range(L + 1):
        assert np.array_equal(st.b(l), ref["b"][l]), f"b level {l}"
        assert np.array_equal(st.u(l), ref["u"][l]), f"u level {l}"
        if l < L:
            assert np.array_equal(st.w(l), ref["w"][l]), f"w level {l}"
    rep = s.error_estimate(1, K.UNSCALED)
    oe = O.estimate3d(ref)
    for a, b in ((rep.norm_base, oe["norm_base"]), (rep.norm_coarser, oe["norm_coarser"]),
                 (rep.conv_factor, oe["conv"]), (rep.eta, oe["eta"])):
        assert abs(a - b) <= 1e-12 * abs(b)
    assert np.max(np.abs(rep.eta_local - oe["local_base"]) / np.maximum(oe["local_base"], 1e-300)) <= 1e-10


@pytest.mark.gpu
def test_fmg_device_source_close_to_faithful():
    """Fast mode (f evaluated with device libm) stays within 1e-9 of the faithful solve."""
    mesh = kuhn_cube(2)
    h = K.GridHierarchy.build(mesh, 4)
    a = K.MultigridSolver(h, K.Problem(K.PROBLEM_SIN3D), K.SolverConfig(nu=2, faithful_source=1)).fmg().u(4)
    b = K.MultigridSolver(h, K.Problem(K.PROBLEM_SIN3D), K.SolverConfig(nu=2, faithful_source=0)).fmg().u(4)
    assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(a))


@pytest.mark.gpu
@pytest.mark.parametrize("name,L", [("kuhn1", 5), ("kuhn1", 6), ("perturbed", 5)])
def test_gauss_seidel_large_levels_bitwise(name, L):
    """The plane-pipelined interior phase (levels with 16 <= n <= 64) against the
    oracle's colour-by-colour sweep: two calls of two sweeps, bit for bit."""
    mesh = kuhn_cube(1) if name == "kuhn1" else _perturbed_kuhn()
    o = O.Hier3D(mesh.coords, mesh.elements, L)
    h = K.GridHierarchy.build(mesh, L)
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_ZERO), K.SolverConfig(nu=2))
    X = o.coords(L)
    x, bb = _smooth(X, 31), _smooth(X, 32)
    gu, gb = K.GridFunction(h, L, x), K.GridFunction(h, L, bb)
    ref = x
    for _ in range(2):
        s.gauss_seidel(gu, gb, 2)
        ref = o.gauss_seidel(L, ref, bb, 2)
        assert np.array_equal(gu.numpy(), ref)
