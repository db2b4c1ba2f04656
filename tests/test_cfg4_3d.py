"""BASELINE.json config 4 (3-d AMR, Gaussian peak): meshes of the reference's
own refine_rg_3d driven by the builder's 3-d oracle (tests/gen_golden_cfg4.py).

Per AMR step k = 0..4 the fixture holds eta, the local indicators eta_T and the
>= 0.5 max marks on the green-reverted set.  The GPU path must reproduce the
indicators (1e-9, BASELINE.json north_star) and the identical marked set.
"""
import json
import os

import numpy as np
import pytest

from _golden import path
from oracle import oracle as O
from paper_2508_06049_b200 import klref as K


def meta():
    with open(path("cfg4.json")) as fh:
        return json.load(fh)


def mesh(k):
    return K.MacroMesh.read(path(f"cfg4_k{k}.mesh"))


def test_cfg4_hierarchies_match_fixture():
    m = meta()
    for k, st in enumerate(m["steps"]):
        h = K.GridHierarchy.build(mesh(k), m["level"], device=False)
        assert h.num_macros() == st["num_macros"]
        assert h.dof_count(m["level"]) == st["dofs"]


def test_cfg4_host_marking_matches_reference():
    """klref_mark (reversion aggregate + 0.5 max rule) on the fixture's indicators."""
    for st in meta()["steps"][:-1]:
        marks = K.mark(K.MARK_HALF_MAX, 0.0, st["active_ids"], st["green_parent"], st["eta_local"],
                       st["reverted_ids"])
        assert marks == st["marks_halfmax_eta"]


def test_cfg4_oracle_pinned_k0():
    m = meta()
    st = m["steps"][0]
    mm = mesh(0)
    o = O.Hier3D(mm.coords, mm.elements, m["level"])
    ref = O.fmg3d(o, "gauss", nu=m["nu"])
    e = O.estimate3d(ref)
    assert abs(e["eta"] - st["eta"]) <= 1e-14 * st["eta"]
    assert np.max(np.abs(e["local_base"] - st["eta_local"])) <= 1e-14 * max(st["eta_local"])


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_cfg4_gpu_estimates_and_marks(k):
    """Faithful f (host-tabulated, the fixture's arithmetic): the FMG state is the
    oracle's bit for bit, so eta agrees to 1e-12 and eta_T elementwise to 1e-10
    (the per-macro sums are reduced in another order); the marks are identical."""
    m = meta()
    st = m["steps"][k]
    h = K.GridHierarchy.build(mesh(k), m["level"])
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_GAUSS3D), K.SolverConfig(nu=m["nu"], faithful_source=1))
    s.fmg()
    rep = s.error_estimate(1, K.UNSCALED)
    assert abs(rep.eta - st["eta"]) <= 1e-12 * st["eta"]
    ref_loc = np.asarray(st["eta_local"])
    assert np.max(np.abs(rep.eta_local - ref_loc) / ref_loc) <= 1e-10
    if "marks_halfmax_eta" in st:
        marks = K.mark(K.MARK_HALF_MAX, 0.0, st["active_ids"], st["green_parent"], rep.eta_local, st["reverted_ids"])
        assert marks == st["marks_halfmax_eta"]


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 4])
def test_cfg4_gpu_device_source_within_tolerance(k):
    """The bench mode (f from device libm): eta and every eta_T within 1e-9 of the
    fixture (BASELINE.json north_star), identical marks."""
    m = meta()
    st = m["steps"][k]
    h = K.GridHierarchy.build(mesh(k), m["level"])
    s = K.MultigridSolver(h, K.Problem(K.PROBLEM_GAUSS3D), K.SolverConfig(nu=m["nu"], faithful_source=0))
    s.fmg()
    rep = s.error_estimate(1, K.UNSCALED)
    assert abs(rep.eta - st["eta"]) <= 1e-9 * st["eta"]
    ref_loc = np.asarray(st["eta_local"])
    assert np.max(np.abs(rep.eta_local - ref_loc) / ref_loc) <= 1e-9
    if "marks_halfmax_eta" in st:
        marks = K.mark(K.MARK_HALF_MAX, 0.0, st["active_ids"], st["green_parent"], rep.eta_local, st["reverted_ids"])
        assert marks == st["marks_halfmax_eta"]
