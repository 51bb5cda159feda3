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
