"""Pins the C restatement oracle (oracle/klref_oracle.c) to the reference itself:
every output must equal the patched reference's (tests/golden, produced by
oracle/_ref/ref_driver) bit for bit — FMG state hashes, single operations,
estimator scalars and local indicators."""
import numpy as np
import pytest

from _golden import golden, npz, path, sha
from _rng import splitmix_uniform
from oracle import oracle as O
from paper_2508_06049_b200.klref import MacroMesh

OPS = [("cfg1", "cfg1.mesh"), ("cfg2k3", "cfg2_k3.mesh")]


@pytest.mark.parametrize("name,mesh", OPS)
def test_oracle_single_operations_bitwise(name, mesh):
    g = golden()["ops_" + name]
    data = npz(f"ops_{name}.npz")
    h = O.Hier2D(MacroMesh.read(path(mesh)), g["L"])
    start = 0
    for l in range(g["L"] + 1):
        N = h.size(l)
        x = h.interface_sync(l, splitmix_uniform(g["seed"], start, N), False)
        bb = h.interface_sync(l, splitmix_uniform(g["seed"], start + N, N), False)
        start += 2 * N
        hs = g["sha256"]
        assert sha(x) == hs[f"x_{l}"] and sha(bb) == hs[f"bb_{l}"]
        assert sha(h.apply(l, x)) == hs[f"Ax_{l}"]
        assert sha(h.apply(l, x, mass=True)) == hs[f"Mx_{l}"]
        assert sha(h.residual(l, x, bb)) == hs[f"res_{l}"]
        assert h.dot_unique(l, x, bb) == float(data[f"dot_{l}"][0])
        if l >= 1:
            u1 = h.gauss_seidel(l, x, bb, 1)
            assert sha(u1) == hs[f"gs1_{l}"]
            assert sha(h.gauss_seidel(l, u1, bb, 1)) == hs[f"gs2_{l}"]
            assert sha(h.restrict(l, x)) == hs[f"restrict_{l}"]
        if l < g["L"]:
            assert sha(h.prolongate(l, x)) == hs[f"prolong_{l}"]
        if l == 0:
            u0, st, _ = h.cg_level0(np.zeros(N), bb)
            assert st == 0 and np.array_equal(u0, data["cg0"])


def _check_state(st, rec, L):
    for l in range(L + 1):
        assert sha(st["u"][l]) == rec["sha256"][f"u_{l}"], f"u level {l}"
        assert sha(st["b"][l]) == rec["sha256"][f"b_{l}"], f"b level {l}"
        if l < L:
            assert sha(st["w"][l]) == rec["sha256"][f"w_{l}"], f"w level {l}"
    for j in range(1, L):
        for kind, tag in ((0, "u"), (1, "s")):
            e = O.estimate2d(st, j, kind)
            assert [e["norm_base"], e["norm_coarser"], e["conv"], e["eta"]] == rec[f"est_{tag}{j}"]
            assert list(e["eta_local"]) == rec[f"eta_local_{tag}{j}"]


def test_oracle_fmg_config1():
    rec = golden()["cfg1"]
    st = O.fmg2d(MacroMesh.read(path("cfg1.mesh")), 6, problem="sin", nu=1)
    assert st["status"] == 0
    _check_state(st, rec, 6)


@pytest.mark.parametrize("k", range(6))
def test_oracle_fmg_config2_amr(k):
    rec = golden()["cfg2"][k]
    mesh = MacroMesh.read(path(f"cfg2_k{k}.mesh"))
    st = O.fmg2d(mesh, 7, problem="lshape", nu=2)
    assert st["hier"].dofs(7) == rec["dofs"]
    _check_state(st, rec, 7)
