"""Parametric B-spline boundary curves (drop-in for wqbem/geometry.py:41-114,
299-327).

The curve is evaluated on the host through scipy ``BSpline`` exactly as the
reference does (geometry.py:83-99), once per quadrature node, so the node
coordinates and speeds fed to the GPU kernels are bit-identical to the ones
the reference's K1 grid sees.  The O(n_q^2) kernel grid itself
(geometry.py:225-248) is evaluated only on the GPU (csrc/wq_ik1.cu).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
from scipy.interpolate import BSpline

from .errors import ConstructionError, GeometryError
from .splines import BasisSpec, as_basis, make_cyclic_basis, make_open_basis

__all__ = ["BoundaryCurve", "as_curve", "curve_eval", "parametric_speed", "load_curve"]

_J_SAMPLES = 1000


@dataclass(frozen=True)
class BoundaryCurve:
    """f(s) = sum_i Q_i B_i(s); cyclic repetition applied internally on
    closed curves (geometry.py:41-80)."""

    basis: BasisSpec
    control_points: np.ndarray

    def __post_init__(self):
        basis = as_basis(self.basis)
        object.__setattr__(self, "basis", basis)
        q = np.asarray(self.control_points, dtype=float)
        object.__setattr__(self, "control_points", q)
        if q.ndim != 2 or q.shape[1] != 2:
            raise ConstructionError("control points must be an (n, 2) array")
        if q.shape[0] != basis.dim:
            raise ConstructionError(
                f"{q.shape[0]} control points for a dimension-{basis.dim} basis")
        coeffs = np.vstack([q, q[: basis.wrap]]) if basis.closed else q
        object.__setattr__(self, "_coeffs", coeffs)
        object.__setattr__(self, "_splines", {0: BSpline(basis.knots, coeffs, basis.degree,
                                                          extrapolate=False)})
        s = np.linspace(basis.a, basis.b, _J_SAMPLES)
        if parametric_speed(self, s).min() <= 0.0:
            raise GeometryError("parametrization is not regular (J <= 0)")

    @property
    def closed(self) -> bool:
        return self.basis.closed

    @property
    def length(self) -> float:
        return self.basis.length

    def is_c2(self) -> bool:
        return self.basis.min_smoothness() >= 2

    def spline(self, deriv_order: int) -> BSpline:
        cache = self._splines
        while deriv_order not in cache:
            k = max(cache)
            cache[k + 1] = cache[k].derivative()
        return cache[deriv_order]


def as_curve(obj) -> BoundaryCurve:
    """Accept this package's curve or the reference's ``BoundaryCurve``."""
    if isinstance(obj, BoundaryCurve):
        return obj
    try:
        return BoundaryCurve(basis=as_basis(obj.basis), control_points=obj.control_points)
    except AttributeError as exc:  # pragma: no cover - defensive
        raise ConstructionError(f"not a boundary curve: {obj!r}") from exc


def _eval_clipped(curve: BoundaryCurve, s, deriv_order: int):
    b = curve.basis
    return curve.spline(deriv_order)(np.clip(np.asarray(s, float), b.a, b.b))


def curve_eval(curve, s, deriv_order: int = 0) -> np.ndarray:
    """f (or a derivative) at s, shape (..., 2) (geometry.py:102-108)."""
    curve = as_curve(curve)
    pts = np.atleast_1d(curve.basis._check_domain(s)).astype(float)
    out = curve.spline(deriv_order)(pts)
    if np.ndim(s) == 0:
        return out[0]
    return out


def parametric_speed(curve, s) -> np.ndarray:
    """J(s) = ||f'(s)|| (geometry.py:111-114)."""
    return np.linalg.norm(curve_eval(curve, s, 1), axis=-1)


def load_curve(source) -> BoundaryCurve:
    """Curve from a JSON path/file or dict (geometry.py:299-327)."""
    if isinstance(source, (str, bytes)) or hasattr(source, "read"):
        if hasattr(source, "read"):
            data = json.load(source)
        else:
            with open(source) as fh:
                data = json.load(fh)
    else:
        data = dict(source)
    degree = int(data["degree"])
    closed = bool(data.get("closed", False))
    if "knots" in data:
        basis = BasisSpec(degree=degree, knots=np.asarray(data["knots"], float), closed=closed)
    elif "breakpoints" in data:
        if closed:
            basis = make_cyclic_basis(degree, data["breakpoints"])
        else:
            basis = make_open_basis(degree, data["breakpoints"], data.get("multiplicities"))
    else:
        raise ConstructionError("curve input needs 'knots' or 'breakpoints'")
    return BoundaryCurve(basis=basis, control_points=data["control_points"])
