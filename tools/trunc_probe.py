"""Probe: how far does dropping the Chebyshev tail of u (splines.cheb_truncated_coeffs)
move A against the reference goldens?  (GPU; tools only.)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import _cases as CS
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as A, splines as S

def patch(disc, tol):
    lp = A._log_part(disc)
    space = disc.space
    curve = disc.curve
    cb = curve.basis
    jac = lambda pts: np.linalg.norm(curve.spline(1)(np.clip(pts, cb.a, cb.b)), axis=-1)
    fine = disc.refined.basis
    u, ucols, D = S.cheb_truncated_coeffs(space, fine.elements, lp.da, scale_fn=jac, tol=tol)
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
