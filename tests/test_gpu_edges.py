"""Partial edge tiles of the closed-uniform fast path: N >= the
x2 kernel's bulk-copy threshold (ZROWS rows of the Z' table) with N % 64 != 0,
so the TMA window path runs together with the cp.async IK1 tile (zero fill),
the non-bulk output stores and the `row < nc` masks on the S band.  Checked
against the oracle (dense restatement at N = 200, row-block restatement at
N = 1000 and 2250) and through every entry point that launches those tiles.
At N = 2250 (666 tile pairs) the single launch runs the warp-specialised
persistent x2 kernel with a partial last tile, the chunked and per-rank
launches the one-pair-per-CTA kernel: they must give the same bits."""

import numpy as np
import pytest

import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS
from _cases import rel

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _ellipse():
    th = 2 * np.pi * np.arange(16) / 16
    return W.load_curve({"degree": 3, "closed": True, "breakpoints": np.linspace(0, 1, 17).tolist(),
                         "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})


def _oracle_A(curve, space, N):
    from oracle import wq_oracle as O
    oc = O.Curve(curve.basis, curve.control_points)
    ob = O.Basis(space.degree, space.knots, space.closed)
    if N <= 256:
        od = O.build_discretization(oc, ob, 1)
        return O.scale_and_symmetrize(O.dense_ik1(od) + O.dense_ik2(od))[0], None
    rows = np.array([0, 1, 63, 64, N // 2, N - 65, N - 2, N - 1])
    return O.CirculantRows(oc, ob).a_rows(rows), rows


@pytest.mark.parametrize("p", [2, 3, 4, 5])
@pytest.mark.parametrize("N", [200, 1000, 2250])
def test_partial_edge_tiles(cuda, p, N):
    torch = cuda
    from paper_1703_10016_b200 import _lib, distributed as D
    curve = _ellipse()
    space = W.make_cyclic_basis(p, np.linspace(0, 1, N + 1))
    disc = W.build_discretization(curve, space, 1)
    assert AS._use_v2(disc) and N % 64 != 0
    A = AS.assemble_matrix_device(disc)
    ref, rows = _oracle_A(curve, space, N)
    got = A.cpu().numpy()
    scale = np.abs(got).max()
    if rows is None:
        assert rel(got, ref) <= TOL
    else:
        assert np.abs(got[rows] - ref).max() / scale <= TOL
    assert np.array_equal(got, got.T)
    # chunked two-stream pipeline: same tiles, same bits
    X = torch.full((N, N), float("nan"), dtype=torch.float64, device="cuda")
    AS._assemble_v2(disc, X, -1.0 / (4 * np.pi), chunks=5)
    torch.cuda.synchronize()
    assert torch.equal(X, A)
    # symmetric multi-GPU path (packed upper tiles), three ranks emulated in turn
    from test_gpu_parity import emulate_packed_ranks
    bufs, _ = emulate_packed_ranks(disc, 3, 2)
    assert all(torch.equal(B, A) for B in bufs)
    # unsymmetrised row blocks (rect tiles) + epilogue
    bounds, per = D.row_blocks(N, 2)
    Xr = torch.zeros((per * 2, N), dtype=torch.float64, device="cuda")
    for r0, r1 in bounds:
        if r1 > r0:
            D.assemble_rows_device(disc, Xr[r0:], r0, r1)
    Ar = Xr[:N].contiguous()
    _lib.call("wq_symmetrize", _lib.ptr(Ar), N, -1.0 / (4 * np.pi), _lib.stream_handle())
    assert rel(Ar.cpu().numpy(), got) <= 1e-14
    # streamed host path
    out = W.assemble_matrix_to_host(disc, chunks=3)
    assert torch.equal(out, A.cpu())
