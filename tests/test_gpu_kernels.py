"""GPU unit tests of kernel building blocks (through the C-ABI self-test hooks)."""

import numpy as np
import pytest

from paper_1703_10016_b200 import _lib

pytestmark = pytest.mark.gpu


def test_fast_half_ln_matches_libdevice(cuda):
    torch = cuda
    rng = np.random.default_rng(0)
    x = np.concatenate([np.exp(rng.uniform(-30, 30, 200000)), 1 + rng.uniform(-1e-3, 1e-3, 50000),
                        [1.0, 2.0, 0.5, 4.0 - 1e-15, 1 + 2 ** -52, 1e-300, 1e300]])
    xd = torch.from_numpy(x).cuda()
    fast, ref = torch.empty_like(xd), torch.empty_like(xd)
    _lib.call("wq_selftest_log", len(x), _lib.ptr(xd), _lib.ptr(fast), _lib.ptr(ref), _lib.stream_handle())
    f, r = fast.cpu().numpy(), ref.cpu().numpy()
    err = np.abs(f - r) / np.maximum(np.abs(r), 1.0)
    assert err.max() <= 4.5e-16, err.max()
    exact = 0.5 * np.log(x)
    assert (np.abs(f - exact) / np.maximum(np.abs(exact), 1.0)).max() <= 4.5e-16


def test_dmma_fragment_layout(cuda):
    torch = cuda
    rng = np.random.default_rng(1)
    A = rng.standard_normal((8, 4))
    B = rng.standard_normal((4, 8))
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = torch.zeros((8, 8), dtype=torch.float64, device="cuda")
    _lib.call("wq_selftest_dmma", _lib.ptr(Ad), _lib.ptr(Bd), _lib.ptr(C), _lib.stream_handle())
    assert np.allclose(C.cpu().numpy(), A @ B, rtol=1e-15, atol=1e-15)


def _general_case(closed: bool):
    """A small general-path discretization (open slit with double knots / closed non-circulant)."""
    import paper_1703_10016_b200 as W
    if closed:
        th = 2 * np.pi * np.arange(16) / 16
        curve = W.load_curve({"degree": 3, "closed": True, "breakpoints": np.linspace(0, 1, 17).tolist(),
                              "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})
        space = W.make_cyclic_basis(3, np.linspace(0, 1, 201))
        return W.build_discretization(curve, space, 2)      # nref = 2: not circulant
    curve = W.load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
    bp = np.linspace(-1, 1, 151)
    mult = np.ones(149, dtype=int)        # interior knots
    mult[[7, 40, 41, 99]] = 2
    space = W.make_open_basis(4, bp, multiplicities=mult)
    return W.build_discretization(curve, space, 1)


@pytest.mark.parametrize("closed", [False, True])
def test_fused_general_kernels_match_unfused(cuda, closed):
    """wq_gather_yts against wq_transpose + wq_gather_fs, and wq_st_phi_sym against
    wq_add_st_phi + wq_symmetrize, on random operands with a real S band (bit-identical
    gathers; the fused symmetrisation to rounding)."""
    torch = cuda
    from paper_1703_10016_b200 import assembly as AS
    disc = _general_case(closed)
    lp, d = AS._logpart_dev(disc)
    assert lp.path == "general"
    N, NE = disc.space.dim, disc.refined.basis.dim
    st = _lib.stream_handle()
    g = torch.Generator(device="cuda").manual_seed(3)
    Y = torch.randn((NE, NE), dtype=torch.float64, device="cuda", generator=g)
    P0 = torch.randn((NE, N), dtype=torch.float64, device="cuda", generator=g)
    # gather: P <- 2 P - Y^T S
    YT = torch.empty_like(Y)
    _lib.call("wq_transpose", _lib.ptr(Y), NE, NE, _lib.ptr(YT), st)
    Pa, Pb = P0.clone(), P0.clone()
    _lib.call("wq_gather_fs", AS.ctypes_ref(d["struct"]), 2.0, _lib.ptr(YT), _lib.ptr(Pa), st)
    _lib.call("wq_gather_yts", AS.ctypes_ref(d["struct"]), 2.0, _lib.ptr(Y), _lib.ptr(Pb),
              AS._s_band_span(lp), st)
    assert torch.equal(Pa, Pb)
    # S^T Phi + symmetrise, with and without an accumulated X
    X0 = torch.randn((N, N), dtype=torch.float64, device="cuda", generator=g)
    for acc in (0, 1):
        Xa, Xb = X0.clone(), X0.clone()
        _lib.call("wq_add_st_phi", AS.ctypes_ref(d["struct"]), _lib.ptr(Pa), 0, N, _lib.ptr(Xa), N, acc, st)
        _lib.call("wq_symmetrize", _lib.ptr(Xa), N, -0.25, st)
        _lib.call("wq_st_phi_sym", AS.ctypes_ref(d["struct"]), _lib.ptr(Pa), _lib.ptr(Xb), -0.25, acc, st)
        a, b = Xa.cpu().numpy(), Xb.cpu().numpy()
        assert np.abs(a - b).max() <= 1e-14 * np.abs(a).max(), acc
        assert np.array_equal(b, b.T)
