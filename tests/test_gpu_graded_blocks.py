"""GPU: the graded-mesh element-pair blocks (wq_gen_pair_blocks: gap-table,
Gauss and near kernels) against the restatement's per-pair moments contracted
the same way, block by block and by pair category."""

import numpy as np
import pytest

import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib
from oracle import wq_oracle as O

pytestmark = pytest.mark.gpu


def _c5like():
    sp = O.config5_space(n_el=96, growth_elems=12)
    slit = W.load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
    return slit, W.BasisSpec(sp.degree, sp.knots, False)


@pytest.mark.parametrize("table", [True, False])
def test_pair_blocks_match_restatement(cuda, table):
    torch = cuda
    curve, space = _c5like()
    disc = W.build_discretization(curve, space, 1)
    lp, d = AS._logpart_dev(disc)
    n = lp.n_el
    nU, nB = lp.u.shape[2], lp.db + 1
    wt = torch.full((n, nU, nB, n), np.nan, dtype=torch.float64, device="cuda")   # [f][a][b][e]
    wd = torch.full((n, nB, nB, n), np.nan, dtype=torch.float64, device="cuda")
    flags = torch.empty((n, -(-n // 64)), dtype=torch.int32, device="cuda")
    m2u = AS._gap_table(disc, lp, 1.0) if table else None
    _lib.call("wq_gen_pair_blocks", n, 0, n, lp.da, lp.db, nU - 1, 0, 0.0,
              _lib.ptr(d["elh"]), _lib.ptr(d["elm"]), _lib.ptr(d["u"]), _lib.ptr(d["v"]),
              _lib.ptr(d["near_lo"]), _lib.ptr(d["near_cnt"]), int(lp.near_cnt.max()),
              _lib.ptr(d["near_unit"]), _lib.ptr(d["touch"]), _lib.ptr(d["gx"]), _lib.ptr(d["gw"]),
              _lib.ptr(m2u) if m2u is not None else None, _lib.ptr(d["ca"]), _lib.ptr(d["cb"]),
              _lib.ptr(wt), _lib.ptr(wd), n, _lib.ptr(flags), _lib.stream_handle())
    wt = wt.cpu().numpy().transpose(3, 0, 1, 2)   # -> [e][f][a][b]
    wd = wd.cpu().numpy().transpose(3, 0, 1, 2)
    e_idx = np.repeat(np.arange(n), n)
    f_idx = np.tile(np.arange(n), n)
    m2 = O.pair_moments_general(lp.da, lp.db, lp.elh[e_idx], lp.elh[f_idx],
                                lp.elm[e_idx] - lp.elm[f_idx]).reshape(n, n, lp.da + 1, nB)
    ref_t = np.einsum("eap,efab,fbq->efpq", lp.u, m2, lp.v)
    ref_d = np.einsum("eap,efab,fbq->efpq", lp.v, m2[:, :, :nB], lp.v)
    h = lp.elh
    rho = h[None, :] / h[:, None]
    delta = lp.elm[:, None] - lp.elm[None, :]
    sep = np.abs(delta) - 0.5 * (h[:, None] + h[None, :])
    near = sep <= 1e-9 * np.maximum(h[:, None], h[None, :])
    same = np.abs(rho - 1) < 1e-10
    cats = {"near equal": near & same, "near unequal": near & ~same, "far equal": ~near & same,
            "far unequal": ~near & ~same}
    scale_t, scale_d = np.abs(ref_t).max(), np.abs(ref_d).max()
    msg = []
    for k, m in cats.items():
        if not m.any():
            continue
        et = np.abs(wt[m] - ref_t[m]).max() / scale_t
        ed = np.abs(wd[m] - ref_d[m]).max() / scale_d
        msg.append(f"{k}: {m.sum()} pairs, theta {et:.2e}, D {ed:.2e}")
    err = np.abs(wt - ref_t).max(axis=(2, 3)) / scale_t
    bad = np.argwhere(err > 1e-12)
    if len(bad):
        msg.append(f"{len(bad)} bad pairs, e.g. {bad[:6].tolist()} widths {h[bad[0][0]]:.6e} {h[bad[0][1]]:.6e}")
    print("\n".join(msg))
    assert np.isfinite(wt).all() and np.isfinite(wd).all()
    assert np.abs(wt - ref_t).max() / scale_t <= 1e-12, msg
    assert np.abs(wd - ref_d).max() / scale_d <= 1e-12, msg
