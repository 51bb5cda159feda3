"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container only (the reference tree does not travel to the
GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Every fixture is produced through the reference's public entry points
(``wqbem.assembly``: build_discretization / assemble_ik1 / assemble_ik2 /
assemble_weighted_matrix / scale_and_symmetrize / assemble_b1 /
assemble_b1_weighted / assemble_b2, assembly.py:147-343) plus, for the
component pins, ``wqbem.quadrature.uniform_pair_log_moments``
(quadrature.py:472) and ``wqbem.splines.local_basis_coeffs``
(splines.py:427).  Small cases store full matrices; larger cases store a
row subset, the diagonal, row sums and norms (size-independent checks).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))

import wqbem  # noqa: E402  (PYTHONPATH must point at the reference)
from wqbem import assembly as A  # noqa: E402
from wqbem.geometry import load_curve  # noqa: E402
from wqbem.splines import make_cyclic_basis, make_open_basis, local_basis_coeffs  # noqa: E402
from wqbem.quadrature import uniform_pair_log_moments  # noqa: E402
from wqbem import problems as P  # noqa: E402

FULL_MAX = 300          # store full matrices up to this dimension
SUBSET_ROWS = (0, 1, 2, 3, 7, 100)


def slit_curve():
    return load_curve({"degree": 1, "knots": [-1, -1, 1, 1],
                       "control_points": [[-1, 0], [1, 0]]})


def ellipse_curve():
    th = 2 * np.pi * np.arange(16) / 16
    return load_curve({"degree": 3, "closed": True,
                       "breakpoints": np.linspace(0, 1, 17).tolist(),
                       "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})


def star_curve():
    th = 2 * np.pi * np.arange(32) / 32
    r = 1 + 0.3 * np.cos(5 * th)
    return load_curve({"degree": 3, "closed": True,
                       "breakpoints": np.linspace(0, 1, 33).tolist(),
                       "control_points": np.column_stack([r * np.cos(th), r * np.sin(th)]).tolist()})


def curve_dict(curve):
    b = curve.basis
    return {"degree": int(b.degree), "knots": b.knots.tolist(), "closed": bool(b.closed),
            "control_points": np.asarray(curve.control_points).tolist()}


def space_dict(space):
    return {"degree": int(space.degree), "knots": space.knots.tolist(), "closed": bool(space.closed)}


class RecordingDatum:
    """Wraps a problem-defined Dirichlet datum (problems.py:48-150) and records
    every (s, u_D(s)) the reference evaluates, so the GPU tests can replay the
    reference's own values as a tabulated datum (the problem code stays in the
    reference)."""

    def __init__(self, fn):
        self.fn, self.pts, self.vals = fn, [], []

    def __call__(self, s):
        v = np.asarray(self.fn(s), dtype=float)
        self.pts.append(np.atleast_1d(np.asarray(s, float)).ravel().copy())
        self.vals.append(np.atleast_1d(v).ravel().copy())
        return v

    def table(self):
        pts = np.concatenate(self.pts)
        vals = np.concatenate(self.vals)
        pts, idx = np.unique(pts, return_index=True)
        return pts, vals[idx]


def run_case(name, curve, space, dirichlet=None, dname=None, b2=False, out=None, nref=1):
    t0 = time.time()
    tabulate = dname in ("parabola", "closed-smooth")
    if tabulate:
        dirichlet = RecordingDatum(dirichlet)
    disc = A.build_discretization(curve, space, nref)
    tb = time.time() - t0
    ik1 = A.assemble_ik1(disc)
    ik2 = A.assemble_ik2(disc)
    m, counters, secs = A.assemble_weighted_matrix(disc)
    a, defect = A.scale_and_symmetrize(m)
    n = space.dim
    rec = {
        "meta": json.dumps({"name": name, "curve": curve_dict(curve), "space": space_dict(space),
                            "nref": nref, "dirichlet": dname, "kernel_evals": counters["kernel_evals"],
                            "defect": defect, "nq": disc.nodes.n, "build_s": tb, "asm_s": secs,
                            "numpy": np.__version__, "scipy": scipy.__version__,
                            "wqbem": wqbem.__version__}),
        "nodes": disc.nodes.nodes,
        "J_nodes": disc.J_nodes,
    }
    if n <= FULL_MAX:
        rec.update(ik1=ik1, ik2=ik2, M=m, A=a, G=disc.G)
    else:
        rows = np.array(sorted({r % n for r in SUBSET_ROWS + (n // 2, n - 1)}))
        rec.update(rows=rows, A_rows=a[rows], M_rows=m[rows], ik1_rows=ik1[rows],
                   A_diag=np.diag(a).copy(), A_rowsum=a.sum(axis=1), A_absmax=np.abs(a).max(),
                   A_fro=np.linalg.norm(a), ik1_diag=np.diag(ik1).copy())
    if dirichlet is not None:
        rec["b1w"] = A.assemble_b1_weighted(disc, dirichlet)
        rec["b1"] = A.assemble_b1(curve, space, dirichlet)
        if b2:
            rec["b2"] = A.assemble_b2(curve, space, dirichlet)
        if tabulate:
            rec["g_pts"], rec["g_vals"] = dirichlet.table()
    if out is not None:
        out.update(rec)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
    print(f"{name}: N={n} nq={disc.nodes.n} build={tb:.2f}s asm={secs:.2f}s defect={defect:.2e}",
          flush=True)
    return disc


def main(which=None):
    from wqbem.assembly import _CurveEval
    slit = slit_curve()
    ell = ellipse_curve()
    star = star_curve()

    def sq(s):
        return np.asarray(s, float) ** 2

    def one(s):
        return np.ones_like(np.asarray(s, float))

    ce_ell = _CurveEval(ell)
    ce_star = _CurveEval(star)

    def g_ell(s):
        f = ce_ell.f(np.asarray(s, float))
        return np.exp(f[:, 0]) * np.cos(f[:, 1])

    def g_star(s):
        f = ce_star.f(np.asarray(s, float))
        return f[:, 0] * f[:, 1]

    cases = []
    # config 1 (CPU config): slit, p=2, 64 elements, g = x^2 (= s^2 on the slit)
    cases.append(("c1_slit_p2_n64", slit, make_open_basis(2, np.linspace(-1, 1, 65)), sq, "x^2", False))
    # open slit variants: other degrees, double knots (uniform widths)
    for p in (3, 4, 5):
        cases.append((f"slit_p{p}_n24", slit, make_open_basis(p, np.linspace(-1, 1, 25)), one, "1", False))
    mult = np.ones(23, dtype=int)
    mult[[3, 8, 9, 15]] = 2
    cases.append(("slit_p4_n24_dbl", slit, make_open_basis(4, np.linspace(-1, 1, 25), mult), one, "1", False))
    # config-2 geometry (ellipse 2x1, 16 ctrl pts), p=3 ladder
    for n in (32, 64, 128, 256):
        cases.append((f"ell_p3_n{n}", ell, make_cyclic_basis(3, np.linspace(0, 1, n + 1)), g_ell,
                      "exp(x)cos(y)", n <= 128))
    for p in (2, 4, 5):
        cases.append((f"ell_p{p}_n64", ell, make_cyclic_basis(p, np.linspace(0, 1, 65)), g_ell,
                      "exp(x)cos(y)", False))
    # config-3 geometry (star, 32 ctrl pts, cubic geometry), p = 2..5
    for p in (2, 3, 4, 5):
        cases.append((f"star_p{p}_n128", star, make_cyclic_basis(p, np.linspace(0, 1, 129)), g_star,
                      "x*y", p == 3))
    # config 2 itself (N=1024): subset storage
    cases.append(("c2_ell_p3_n1024", ell, make_cyclic_basis(3, np.linspace(0, 1, 1025)), g_ell,
                  "exp(x)cos(y)", True))
    # config 3 degree sweep at reduced N (N=4096 needs ~35 GB / 10 min per degree in the reference)
    for p in (2, 3, 4, 5):
        cases.append((f"star_p{p}_n512", star, make_cyclic_basis(p, np.linspace(0, 1, 513)), g_star,
                      "x*y", False))
    # reference problems (problems.py)
    par = P.define_problem("parabola")
    for p in (2, 3):
        cases.append((f"parabola_p{p}_n16", par.curve, par.make_space(p, 16), par.dirichlet,
                      "parabola", False))
    cs = P.define_problem("closed-smooth")
    cases.append(("closed_smooth_p3_n24", cs.curve, cs.make_space(3, 24), cs.dirichlet,
                  "closed-smooth", False))

    # config 3 at its stated size (N = 4096): ~10 min and ~35 GB per degree in the
    # reference, so only generated when asked for explicitly ("c3_star")
    for p in (2, 3, 4, 5):
        cases.append((f"c3_star_p{p}_n4096", star, make_cyclic_basis(p, np.linspace(0, 1, 4097)),
                      g_star, "x*y", False))

    for name, curve, space, g, gname, b2 in cases:
        if name.startswith("c3_star") and not (which and any(w in name for w in which)):
            continue
        if which and not any(w in name for w in which):
            continue
        run_case(name, curve, space, g, gname, b2)

    # refined exactness space (nref = 2): closed -> general (non-circulant) path, open too
    for name, curve, space, g, gname in (
            ("ell_p3_n32_nref2", ell, make_cyclic_basis(3, np.linspace(0, 1, 33)), g_ell,
             "exp(x)cos(y)"),
            ("slit_p2_n16_nref2", slit, make_open_basis(2, np.linspace(-1, 1, 17)), sq, "x^2"),
            # the widest rule bands (degree 4 / 5 with nref = 2)
            ("ell_p4_n24_nref2", ell, make_cyclic_basis(4, np.linspace(0, 1, 25)), g_ell,
             "exp(x)cos(y)"),
            ("ell_p5_n128_nref2", ell, make_cyclic_basis(5, np.linspace(0, 1, 129)), g_ell,
             "exp(x)cos(y)"),
            ("slit_p4_n20_nref2", slit, make_open_basis(4, np.linspace(-1, 1, 21)), sq, "x^2"),
            ("slit_p5_n128_nref2", slit, make_open_basis(5, np.linspace(-1, 1, 129)), sq, "x^2")):
        if which and not any(w in name for w in which):
            continue
        run_case(name, curve, space, g, gname, False, nref=2)

    if not which or "components" in which:
        # component pins: pair-moment tables and local polynomial coefficients
        comp = {}
        for tag, sp, curve in (("open", make_open_basis(2, np.linspace(-1, 1, 65)), slit),
                               ("closed", make_cyclic_basis(3, np.linspace(0, 1, 65)), ell)):
            bigd = sp.degree + A._JFIT_DEGREE
            m2, kmap = uniform_pair_log_moments(sp, bigd)
            comp[f"{tag}_m2"] = m2
            comp[f"{tag}_kmap"] = kmap
            u, ucols = local_basis_coeffs(sp, sp.elements, bigd, scale_fn=_CurveEval(curve).jac)
            v, vcols = local_basis_coeffs(sp, sp.elements, sp.degree)
            comp[f"{tag}_u"] = u
            comp[f"{tag}_ucols"] = ucols
            comp[f"{tag}_v"] = v
            comp[f"{tag}_vcols"] = vcols
        # closed ellipse at N=1024 pair table (scaling law at small h)
        sp = make_cyclic_basis(3, np.linspace(0, 1, 1025))
        comp["closed1024_m2"], _ = uniform_pair_log_moments(sp, 15)
        np.savez_compressed(os.path.join(HERE, "components.npz"), **comp)
        print("components written")

    if not which or "naive" in which:
        # the reference's own independent oracles (pkg/tests/oracles.py) on a tiny case
        sys.path.insert(0, "/root/reference/pkg/tests")
        import oracles  # noqa: E402
        sp = make_cyclic_basis(3, np.linspace(0, 1, 13))
        disc = A.build_discretization(ell, sp, 1)
        rec = {"naive_ik1": oracles.naive_ik1(disc), "naive_ik2": oracles.naive_ik2(disc),
               "ik1": A.assemble_ik1(disc), "ik2": A.assemble_ik2(disc),
               "meta": json.dumps({"curve": curve_dict(ell), "space": space_dict(sp)})}
        np.savez_compressed(os.path.join(HERE, "naive_ell_p3_n12.npz"), **rec)
        print("naive written")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
