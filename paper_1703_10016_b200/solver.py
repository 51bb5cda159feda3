"""Dense solve of the assembled system on the device.

Mirrors ``wqbem.solver.solve_system`` (solver.py:60-83) and
``condition_number`` (:86-93): Cholesky first (cuSOLVER potrf/potrs through
torch.linalg), LU with partial pivoting (getrf/getrs) with a RuntimeWarning
when the matrix is not positive definite, SolverError on a singular or
non-finite system or when the relative residual ||A x - b|| / ||b|| exceeds
1e-10.  The matrix may be the device tensor of ``assemble_matrix_device`` (no
host round trip of the N^2 matrix) or a numpy array; the result has the type
of the right-hand side.  No CPU fallback.
"""

from __future__ import annotations

import warnings

import numpy as np

from .errors import DeviceError, SolverError

RESIDUAL_TOL = 1e-10   # solver.py:30


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise DeviceError("PyTorch is required for device memory") from exc
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 solve has no CPU fallback")
    return torch


def _as_dev(torch, x):
    if hasattr(x, "is_cuda") and x.is_cuda:
        return x.to(torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=float))).to("cuda")


def solve_system(matrix, rhs):
    """x with A x = b (solver.py:60-83 semantics)."""
    torch = _torch()
    host_rhs = not (hasattr(rhs, "is_cuda") and rhs.is_cuda)
    A = _as_dev(torch, matrix)
    b = _as_dev(torch, rhs)
    if not (bool(torch.isfinite(A).all()) and bool(torch.isfinite(b).all())):
        raise SolverError("non-finite entries in the linear system")
    vec = b.ndim == 1
    B = b.reshape(-1, 1) if vec else b
    L, info = torch.linalg.cholesky_ex(A)
    if int(info.item()) == 0:
        x = torch.cholesky_solve(B, L)
    else:
        warnings.warn("Cholesky failed (matrix not positive definite); using LU", RuntimeWarning)
        LU, piv, info = torch.linalg.lu_factor_ex(A)
        if int(info.item()) != 0:
            raise SolverError("linear system is singular")
        x = torch.linalg.lu_solve(LU, piv, B)
    scale = float(torch.linalg.norm(B))
    resid = float(torch.linalg.norm(A @ x - B)) / (scale if scale > 0 else 1.0)
    if not np.isfinite(resid) or resid > RESIDUAL_TOL:
        raise SolverError(f"solver residual {resid:.2e} exceeds tolerance")
    x = x.reshape(-1) if vec else x
    return x.cpu().numpy() if host_rhs else x


def condition_number(matrix) -> float:
    """|lambda|_max / |lambda|_min of the symmetrised matrix (solver.py:86-93;
    device syevd)."""
    torch = _torch()
    A = _as_dev(torch, matrix)
    lam = torch.linalg.eigvalsh(0.5 * (A + A.T)).abs()
    lo = float(lam.min())
    return float("inf") if lo == 0.0 else float(lam.max()) / lo
