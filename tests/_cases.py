"""Golden fixture loading shared by the tests (fixtures made by
tests/golden/make_golden.py from the unmodified reference)."""

import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names(kind="all"):
    out = []
    for f in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        name = os.path.basename(f)[:-4]
        if name in ("components",) or name.startswith("naive"):
            continue
        out.append(name)
    return out


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    return z, meta


def product_objects(meta):
    import paper_1703_10016_b200 as W
    c, sp = meta["curve"], meta["space"]
    curve = W.BoundaryCurve(W.BasisSpec(c["degree"], np.array(c["knots"]), c["closed"]),
                            c["control_points"])
    space = W.BasisSpec(sp["degree"], np.array(sp["knots"]), sp["closed"])
    return curve, space


def oracle_objects(meta):
    from oracle import wq_oracle as O
    curve = O.Curve.from_dict(meta["curve"])
    sp = meta["space"]
    return curve, O.Basis(sp["degree"], np.array(sp["knots"]), sp["closed"])


def dirichlet(meta, curve_eval):
    """The Dirichlet datum the fixture was generated with, as u_D(s)."""
    name = meta["dirichlet"]
    if name == "x^2":
        return lambda s: np.asarray(s, float) ** 2
    if name == "1":
        return lambda s: np.ones_like(np.asarray(s, float))
    if name == "exp(x)cos(y)":
        def g(s):
            f = curve_eval(np.asarray(s, float))
            return np.exp(f[:, 0]) * np.cos(f[:, 1])
        return g
    if name == "x*y":
        def g(s):
            f = curve_eval(np.asarray(s, float))
            return f[:, 0] * f[:, 1]
        return g
    return None


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())
