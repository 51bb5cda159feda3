"""GPU: dense solve of the assembled system against the
reference's solve_system semantics (solver.py:60-83): scipy Cholesky/LU on
the same matrices, <= 1e-9 relative on the density coefficients."""

import warnings

import numpy as np
import pytest
import scipy.linalg

import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS
from paper_1703_10016_b200.errors import SolverError
from _cases import load, product_objects, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["ell_p3_n256", "c2_ell_p3_n1024", "slit_p4_n24_dbl"])
def test_solve_matches_scipy_on_golden_systems(cuda, name):
    z, meta = load(name)
    A = z["A"] if "A" in z.files else None
    curve, space = product_objects(meta)
    disc = W.build_discretization(curve, space, meta["nref"])
    Ad = AS.assemble_matrix_device(disc)
    b = z["b1w"] if "b1w" in z.files else np.ones(space.dim)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        x = W.solve_system(Ad, b)                        # device matrix, host rhs
    Ah = Ad.cpu().numpy() if A is None else A
    try:   # the reference's order (solver.py:66-79): Cholesky, else LU
        ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(Ah), b)
    except np.linalg.LinAlgError:    # ellipse 2x1: log capacity 1.5 > 1, A indefinite
        ref = scipy.linalg.solve(Ah, b)
    assert rel(x, ref) <= 1e-9
    assert np.isfinite(W.condition_number(Ad))


def test_lu_fallback_and_errors(cuda):
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.normal(size=(64, 64)))
    A = Q @ np.diag(np.linspace(-1, 2, 64) + 0.01) @ Q.T    # symmetric indefinite
    b = rng.normal(size=64)
    with pytest.warns(RuntimeWarning, match="using LU"):
        x = W.solve_system(A, b)
    assert rel(x, scipy.linalg.solve(A, b)) <= 1e-9
    with pytest.raises(SolverError, match="non-finite"):
        W.solve_system(np.full((4, 4), np.nan), np.ones(4))
    with pytest.raises(SolverError):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            W.solve_system(np.zeros((8, 8)), np.ones(8))
