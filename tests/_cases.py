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


def tabulated(pts, vals):
    """u_D(s) replaying the values the reference computed at exactly these
    parameters (problem-defined data, problems.py:48-150); any other s is a
    test error."""
    pts = np.asarray(pts, float)
    vals = np.asarray(vals, float)

    def g(s):
        s = np.atleast_1d(np.asarray(s, float))
        k = np.clip(np.searchsorted(pts, s), 0, len(pts) - 1)
        km = np.clip(k - 1, 0, len(pts) - 1)
        k = np.where(np.abs(pts[km] - s) < np.abs(pts[k] - s), km, k)
        off = np.abs(pts[k] - s)
        if off.max() > 1e-13 * max(1.0, np.abs(pts).max()):
            raise AssertionError(f"datum requested off the reference's points ({off.max():.2e})")
        return vals[k]
    return g


def dirichlet(meta, curve_eval, z=None):
    """The Dirichlet datum the fixture was generated with, as u_D(s)."""
    name = meta["dirichlet"]
    if z is not None and "g_pts" in z:
        return tabulated(z["g_pts"], z["g_vals"])
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
