"""Effectivity constants, spread bounds and indices (proj/src/estimator.cpp:47-123)
through the C-ABI (klref_effectivity_*), against golden values computed by the
reference itself (tests/gen_golden_effectivity.py) and the paper's C1/C2 table.
Host code: no GPU needed."""
import json
import math
import os

import numpy as np
import pytest

from paper_2508_06049_b200 import klref as K

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "effectivity.json")


def _close(a, b):
    if math.isnan(b):
        return math.isnan(a)
    return a == b or abs(a - b) <= 4e-16 * abs(b)


def test_bounds_match_reference():
    d = json.load(open(GOLD))
    for c in d["bounds"]:
        if c["error"]:
            with pytest.raises(K.DomainError):
                K.make_bounds(c["theta"], c["eps"], c["offset"])
            continue
        b = K.make_bounds(c["theta"], c["eps"], c["offset"])
        lo, up, ss, su, order = c["values"]
        assert _close(b.equivalence.lower, lo) and _close(b.equivalence.upper, up), c
        assert _close(b.spread_scaled, ss) and _close(b.spread_unscaled, su), c
        assert b.order == order


def test_paper_table_constants():
    """C1, C2 of PAPER.md table eff_idx (theta = 2^-q, eps = 0; q = 2 waves, q = 4/3 L-shape)."""
    table = {2.0: [(0.53, 1.67), (0.80, 1.24), (0.93, 1.08), (0.98, 1.02)],
             4.0 / 3.0: [(0.31, 2.32), (0.53, 1.76), (0.72, 1.37), (0.85, 1.18)]}
    for q, rows in table.items():
        for j, (c1, c2) in enumerate(rows, start=1):
            c = K.effectivity_constants(2.0 ** -q, 0.0, j)
            assert round(c.lower, 2) == c1 and round(c.upper, 2) == c2
    b = K.make_bounds_from_order(2, 0.0, 1)
    assert b.order == 2 and b.theta == 0.25


def test_effectivity_index_matches_reference():
    d = json.load(open(GOLD))
    for c in d["effectivity_index"]:
        rep = K.EstimateReport(offset=1, base_level=0, kind=K.UNSCALED, norm_coarser=0.0, norm_base=0.0,
                               conv_factor=0.0, eta=c["eta"], eta_local=np.array(c["eta_local"]))
        e = K.effectivity_index(rep, (c["exact_global"], np.array(c["exact_local"])))
        assert e.gamma_valid == c["gamma_valid"] and e.spread_valid == c["spread_valid"]
        assert _close(e.gamma, c["gamma"]) and _close(e.spread, c["spread"])
        assert len(e.gamma_local) == len(c["gamma_local"])
        for a, b in zip(e.gamma_local, c["gamma_local"]):
            assert _close(a, b)
