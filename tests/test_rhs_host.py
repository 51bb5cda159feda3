"""RHS parity on the CPU side: the oracle's weighted b1w and the product's
host Gauss b1 (assembly.py:287-319) against the reference's goldens, for
every datum -- analytic ones and the problem-defined parabola / closed-smooth
data (problems.py:48-150), which replay the reference's own values."""

import numpy as np
import pytest

import paper_1703_10016_b200 as W
from _cases import dirichlet, golden_names, load, oracle_objects, product_objects, rel

RHS = [n for n in golden_names() if "b1w" in load(n)[0]]


@pytest.mark.parametrize("name", RHS)
def test_b1_host_and_oracle_b1w_match_reference(name):
    from oracle import wq_oracle as O
    z, meta = load(name)
    curve, space = product_objects(meta)
    g = dirichlet(meta, lambda s: W.curve_eval(curve, s), z)
    assert g is not None
    assert rel(W.assemble_b1(curve, space, g), z["b1"]) <= 1e-11
    if space.dim <= 1100:
        oc, ob = oracle_objects(meta)
        od = O.build_discretization(oc, ob, meta["nref"])
        assert rel(O.b1_weighted(od, g), z["b1w"]) <= 1e-11


def test_problem_data_are_tabulated():
    for name in ("parabola_p2_n16", "parabola_p3_n16", "closed_smooth_p3_n24"):
        z, meta = load(name)
        assert "g_pts" in z and len(z["g_pts"]) == len(z["g_vals"]) > 0
