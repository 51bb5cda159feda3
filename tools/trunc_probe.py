"""Probe: how far does dropping the Chebyshev tail of u (splines.cheb_truncated_coeffs)
move A against the reference goldens?  (GPU; tools only.)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import _cases as CS
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as A, splines as S
from scipy.interpolate import BSpline

def cheb_truncated_coeffs(basis, elements, degree, scale_fn=None, tol=1e-11):
    """``local_basis_coeffs`` with the interpolant's Chebyshev tail dropped.

    The reference interpolates B_i(s)·J(s) at ``degree + 1`` Chebyshev points
    and converts with the inverse monomial Vandermonde (splines.py:427-472).
    The interpolant is the same polynomial as sum_k c_k T_k(x) with the
    discrete Chebyshev coefficients c_k of those values; for k above the
    B-spline degree they carry J's variation across one element (decaying
    like (h/curve scale)^k) and then the round-off of the sample positions
    (≈1e-13 of max|c| on fine meshes), which the monomial conversion amplifies
    into coefficients of size ~1e-10 that cancel pointwise.  Terms with
    max|c_k| ≤ tol·max|c| for every k above a cut D are dropped, so the
    polynomial moves pointwise by at most sum_{k>D} |c_k| (the reference's own
    noise level) and its monomial coefficients vanish above D.  The log part
    then contracts only D + 1 powers (``LogPart.na_used``).

    Returns ``(coeffs (n_el, degree+1, basis.degree+1), cols, D)``; coeffs is
    zero in powers > D.
    """
    from numpy.polynomial import chebyshev as npc

    x, _ = S._cheb_setup(degree)
    n = degree + 1
    elements = np.asarray(elements, dtype=float)
    n_el = len(elements)
    half = 0.5 * (elements[:, 1] - elements[:, 0])
    mid = 0.5 * (elements[:, 0] + elements[:, 1])
    pts = (mid[:, None] + half[:, None] * x[None, :]).ravel()
    mat = BSpline.design_matrix(pts, basis.knots, basis.degree)
    width = basis.degree + 1
    if mat.indptr[-1] != len(pts) * width:
        raise ValueError("local interpolation points must lie strictly inside knot spans")
    cols_all = mat.indices.reshape(n_el, n, width)
    if np.any(cols_all[:, 0, :] != cols_all[:, -1, :]):
        raise ValueError("each element must lie inside a single knot span")
    cols = cols_all[:, 0, :].copy()
    if basis.closed:
        cols[cols >= basis.dim] -= basis.dim
    vals = mat.data.reshape(n_el, n, width)
    if scale_fn is not None:
        vals = vals * np.asarray(scale_fn(pts), dtype=float).reshape(n_el, n, 1)
    # discrete Chebyshev transform at the first-kind points (exact orthogonality)
    tk = np.cos(np.outer(np.arange(n), np.arccos(x)))
    c = np.einsum("kj,ejb->ekb", tk, vals) * (2.0 / n)
    c[:, 0] *= 0.5
    prof = np.abs(c).max(axis=(0, 2))
    big = np.nonzero(prof > tol * prof.max())[0]
    D = int(max(big.max() if len(big) else 0, basis.degree))
    conv = np.zeros((D + 1, D + 1))  # conv[k, a]: coefficient of x^a in T_k
    for k in range(D + 1):
        e = np.zeros(k + 1)
        e[k] = 1.0
        conv[k, : k + 1] = npc.cheb2poly(e)
    coeffs = np.zeros((n_el, n, width))
    coeffs[:, : D + 1, :] = np.einsum("ka,ekb->eab", conv, c[:, : D + 1, :])
    coeffs[:, : D + 1, :] *= (half[:, None] ** -np.arange(D + 1)[None, :])[:, :, None]
    return coeffs, cols, D


def patch(disc, tol):
    lp = A._log_part(disc)
    space = disc.space
    curve = disc.curve
    cb = curve.basis
    jac = lambda pts: np.linalg.norm(curve.spline(1)(np.clip(pts, cb.a, cb.b)), axis=-1)
    fine = disc.refined.basis
    u, ucols, D = cheb_truncated_coeffs(space, fine.elements, lp.da, scale_fn=jac, tol=tol)
    n = fine.n_elements; N = space.dim; tu = lp.U.shape[1]
    e_start = np.arange(N) - space.degree
    for a in range(tu):
        e = np.mod(e_start + a, n)
        loc = np.mod(np.arange(N) - e, n)
        lp.U[:, a, :] = u[e, :, loc]
        lp.uext[:, a * lp.nApad: a * lp.nApad + lp.da + 1] = 2.0 * lp.U[:, a, :]
    return D

for tol in [1e-11, 1e-12]:
  for name in CS.golden_names():
    z, meta = CS.load(name)
    if not meta["space"]["closed"] or meta.get("nref", 1) != 1:
        continue
    curve, space = CS.product_objects(meta)
    disc = W.build_discretization(curve, space, 1)
    if A._log_part(disc).path != "circulant":
        continue
    a0, _ = W.scale_and_symmetrize(W.assemble_weighted_matrix(disc)[0])
    disc = W.build_discretization(curve, space, 1)
    D = patch(disc, tol)
    a1, _ = W.scale_and_symmetrize(W.assemble_weighted_matrix(disc)[0])
    if "A_rows" in z.files:
        rows = z["rows"]; ref = z["A_rows"]; s0 = a0[rows]; s1 = a1[rows]; amax = float(z["A_absmax"])
    else:
        ref = z["A"]; s0 = a0; s1 = a1; amax = np.abs(ref).max()
    e0 = np.abs(s0 - ref).max() / amax; e1 = np.abs(s1 - ref).max() / amax
    print(f"tol {tol:.0e} {name:24s} D={D:2d} err_full {e0:.2e} err_trunc {e1:.2e} trunc-vs-full {np.abs(a1-a0).max()/np.abs(a0).max():.2e}", flush=True)

import torch
th = 2 * np.pi * np.arange(16) / 16
ell = W.load_curve({"degree": 3, "closed": True, "breakpoints": np.linspace(0, 1, 17).tolist(),
                    "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})
for n in [4096, 32768]:
    space = W.make_cyclic_basis(3, np.linspace(0, 1, n + 1))
    disc = W.build_discretization(ell, space, 1)
    a0 = A.assemble_matrix_device(disc)
    disc = W.build_discretization(ell, space, 1)
    D = patch(disc, 1e-11)
    a1 = A.assemble_matrix_device(disc)
    d = (a1 - a0).abs().max().item() / a0.abs().max().item()
    print(f"ellipse n={n} D={D} trunc-vs-full {d:.2e}", flush=True)
    del a0, a1
    torch.cuda.empty_cache()
