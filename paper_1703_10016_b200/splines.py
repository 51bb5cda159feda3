"""B-spline spaces on open (clamped) and closed (cyclic) parameter domains.

Drop-in for ``wqbem.splines`` (splines.py:41-257): same class and factory
names, same knot layouts, same validation errors.  Objects from the
reference package are accepted anywhere a ``BasisSpec`` is expected (duck
typing on ``degree`` / ``knots`` / ``closed``).

All evaluation here is vectorised and O(n_points): it feeds the O(N) host
precompute of the GPU assembly (nodes, rule bands, per-element polynomial
coefficients).  Nothing in this module is on the O(N^2) path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property, lru_cache

import numpy as np
from scipy.interpolate import BSpline

from .errors import ConstructionError, DomainError

__all__ = [
    "BasisSpec",
    "RefinedBasis",
    "make_open_basis",
    "make_cyclic_basis",
    "refine_uniform",
    "as_basis",
    "active_values",
    "local_basis_coeffs",
]

_DOMAIN_RTOL = 1e-12


@dataclass(frozen=True)
class BasisSpec:
    """Degree + extended knot vector + open/closed flag (splines.py:41-152)."""

    degree: int
    knots: np.ndarray
    closed: bool = False

    def __post_init__(self):
        knots = np.asarray(self.knots, dtype=float)
        object.__setattr__(self, "knots", knots)
        d = self.degree
        if d < 0:
            raise ConstructionError("degree must be non-negative")
        if knots.ndim != 1 or len(knots) < 2 * d + 2:
            raise ConstructionError("knot vector too short for degree")
        if np.any(np.diff(knots) < 0):
            raise ConstructionError("knots must be non-decreasing")
        if self.nplain < d + 1:
            raise ConstructionError("basis needs at least degree+1 functions")
        if self.closed and self.dim < 1:
            raise ConstructionError("cyclic basis needs dimension >= 1")
        if np.any(self.multiplicities[1:-1] > max(d, 1)):
            raise ConstructionError("inner breakpoint multiplicity exceeds degree")

    @property
    def nplain(self) -> int:
        return len(self.knots) - self.degree - 1

    @property
    def seam_multiplicity(self) -> int:
        tol = _DOMAIN_RTOL * max(float(self.knots[-1] - self.knots[0]), 1.0)
        return int(np.count_nonzero(np.abs(self.knots - self.a) <= tol))

    @property
    def wrap(self) -> int:
        """Plain functions folded onto their periodic images (closed)."""
        return self.degree + 1 - self.seam_multiplicity if self.closed else 0

    @property
    def dim(self) -> int:
        return self.nplain - self.wrap

    @property
    def a(self) -> float:
        return float(self.knots[self.degree])

    @property
    def b(self) -> float:
        return float(self.knots[self.nplain])

    @property
    def length(self) -> float:
        return self.b - self.a

    @cached_property
    def _break(self):
        inner = self.knots[self.degree: self.nplain + 1]
        return np.unique(inner, return_counts=True)

    @property
    def breakpoints(self) -> np.ndarray:
        return self._break[0]

    @property
    def multiplicities(self) -> np.ndarray:
        return self._break[1]

    @cached_property
    def elements(self) -> np.ndarray:
        bp = self.breakpoints
        return np.column_stack([bp[:-1], bp[1:]])

    @property
    def n_elements(self) -> int:
        return len(self.breakpoints) - 1

    def fold(self, plain_index):
        return plain_index if not self.closed else np.mod(plain_index, self.dim)

    def min_smoothness(self) -> int:
        inner = list(self.multiplicities[1:-1])
        if self.closed:
            inner.append(self.seam_multiplicity)
        return self.degree if not inner else self.degree - max(inner)

    def _check_domain(self, s):
        s = np.asarray(s, dtype=float)
        tol = _DOMAIN_RTOL * max(self.length, 1.0)
        if np.any(s < self.a - tol) or np.any(s > self.b + tol):
            raise DomainError(f"point outside parametric domain [{self.a}, {self.b}]")
        return np.clip(s, self.a, self.b)


@dataclass(frozen=True)
class RefinedBasis:
    """Exactness space: each parent element split into nref pieces."""

    parent: BasisSpec
    nref: int
    basis: BasisSpec = field(repr=False)

    @property
    def dim(self) -> int:
        return self.basis.dim


def as_basis(obj) -> BasisSpec:
    """Accept this package's BasisSpec or any duck-typed equivalent (e.g. the
    reference's ``wqbem.splines.BasisSpec``)."""
    if isinstance(obj, BasisSpec):
        return obj
    try:
        return BasisSpec(int(obj.degree), np.asarray(obj.knots, float), bool(obj.closed))
    except AttributeError as exc:  # pragma: no cover - defensive
        raise ConstructionError(f"not a B-spline basis: {obj!r}") from exc


def make_open_basis(degree, breakpoints, multiplicities=None) -> BasisSpec:
    """Clamped basis (splines.py:168-196)."""
    bp = np.asarray(breakpoints, dtype=float)
    if len(bp) < 2 or np.any(np.diff(bp) <= 0):
        raise ConstructionError("need >= 2 strictly increasing breakpoints")
    inner = bp[1:-1]
    if multiplicities is None:
        mult = np.ones(len(inner), dtype=int)
    else:
        mult = np.asarray(multiplicities, dtype=int)
        if len(mult) == len(bp):
            if mult[0] > degree + 1 or mult[-1] > degree + 1:
                raise ConstructionError("end multiplicity exceeds degree+1")
            mult = mult[1:-1]
        elif len(mult) != len(inner):
            raise ConstructionError("multiplicity list does not match breakpoints")
    if np.any(mult < 1) or np.any(mult > degree):
        raise ConstructionError("inner multiplicities must lie in [1, degree]")
    knots = np.concatenate([np.full(degree + 1, bp[0]), np.repeat(inner, mult),
                            np.full(degree + 1, bp[-1])])
    return BasisSpec(degree=degree, knots=knots, closed=False)


def make_cyclic_basis(degree, breakpoints, multiplicities=None) -> BasisSpec:
    """Periodic basis (splines.py:199-236): auxiliary knots are the periodic
    images of the knots next to the opposite end."""
    bp = np.asarray(breakpoints, dtype=float)
    if len(bp) < 3 or np.any(np.diff(bp) <= 0):
        raise ConstructionError("cyclic basis needs >= 3 strictly increasing breakpoints")
    if multiplicities is None:
        mult = np.ones(len(bp), dtype=int)
    else:
        mult = np.asarray(multiplicities, dtype=int)
        if len(mult) != len(bp):
            raise ConstructionError("multiplicity list does not match breakpoints")
        if mult[0] != mult[-1]:
            raise ConstructionError("seam multiplicities must agree")
    if np.any(mult < 1) or np.any(mult > degree):
        raise ConstructionError("cyclic multiplicities must lie in [1, degree]")
    period = bp[-1] - bp[0]
    one = np.repeat(bp[:-1], mult[:-1])
    dim = len(one)
    ms = int(mult[0])
    start = dim + ms - 1 - degree
    if start < 0:
        raise ConstructionError("cyclic basis needs more breakpoints for this degree")
    full = np.concatenate([one - period, one, one + period])
    return BasisSpec(degree=degree, knots=full[start: start + dim + 2 * degree + 2 - ms],
                     closed=True)


def refine_uniform(basis, nref: int) -> RefinedBasis:
    """Split each element into nref equal pieces (splines.py:239-257)."""
    basis = as_basis(basis)
    if nref < 1:
        raise ConstructionError("nref must be >= 1")
    bp = basis.breakpoints
    # np.linspace(lo, hi, nref + 1)[:-1] per element, vectorised with linspace's own
    # arithmetic (k * ((hi - lo) / nref) + lo), so the breakpoints are bit-identical
    lo, hi = bp[:-1], bp[1:]
    step = (hi - lo) / nref
    pieces = np.arange(nref, dtype=float)[None, :] * step[:, None] + lo[:, None]
    nbp = np.concatenate([pieces.ravel(), bp[-1:]])
    nm = np.ones(len(nbp), dtype=int)
    nm[::nref] = basis.multiplicities
    if basis.closed:
        nm[0] = nm[-1] = basis.seam_multiplicity
        fine = make_cyclic_basis(basis.degree, nbp, nm)
    else:
        fine = make_open_basis(basis.degree, nbp, nm)
    return RefinedBasis(parent=basis, nref=nref, basis=fine)


# -- vectorised evaluation ---------------------------------------------------


def active_values(basis: BasisSpec, pts):
    """Values of the degree+1 plain functions of each point's knot span.

    Returns ``(vals, cols)`` of shape (n_pts, degree+1); ``cols`` are FOLDED
    (logical) indices.  Uses scipy's design matrix, i.e. the same evaluation
    the reference's ``basis_values`` uses (assembly.py:101-108).
    """
    pts = np.clip(np.atleast_1d(np.asarray(pts, float)), basis.a, basis.b)
    mat = BSpline.design_matrix(pts, basis.knots, basis.degree)
    width = basis.degree + 1
    if mat.indptr[-1] != len(pts) * width:
        raise ConstructionError("evaluation points produced a ragged design matrix")
    vals = mat.data.reshape(len(pts), width).copy()
    cols = mat.indices.reshape(len(pts), width).copy()
    if basis.closed:
        cols[cols >= basis.dim] -= basis.dim
    return vals, cols


@lru_cache(maxsize=32)
def _cheb_setup(degree: int):
    """Chebyshev points on (-1, 1) and their inverse increasing Vandermonde
    (the reference recipe, splines.py:388-396: np.linalg.inv of np.vander)."""
    x = np.cos(np.pi * (2 * np.arange(degree + 1) + 1) / (2 * degree + 2))
    vinv = np.linalg.inv(np.vander(x, degree + 1, increasing=True))
    x.setflags(write=False)
    vinv.setflags(write=False)
    return x, vinv


def local_basis_coeffs(basis, elements, degree, scale_fn=None):
    """Per-element coefficients of the active functions in powers of
    (s - mid_e), optionally times a smooth factor (splines.py:427-472).

    Same interpolation recipe as the reference (Chebyshev points, cached
    inverse Vandermonde, half^-k scaling) so the coefficient round-off
    matches.  Returns ``(coeffs (n_el, degree+1, basis.degree+1), cols)``.
    """
    basis = as_basis(basis)
    if degree < 0:
        raise ConstructionError("polynomial degree must be non-negative")
    x, vinv = _cheb_setup(degree)
    powers = np.arange(degree + 1)
    elements = np.asarray(elements, dtype=float)
    n_el = len(elements)
    half = 0.5 * (elements[:, 1] - elements[:, 0])
    mid = 0.5 * (elements[:, 0] + elements[:, 1])
    pts = (mid[:, None] + half[:, None] * x[None, :]).ravel()
    mat = BSpline.design_matrix(pts, basis.knots, basis.degree)
    width = basis.degree + 1
    if mat.indptr[-1] != len(pts) * width:
        raise ConstructionError("local interpolation points must lie strictly inside knot spans")
    cols_all = mat.indices.reshape(n_el, degree + 1, width)
    if np.any(cols_all[:, 0, :] != cols_all[:, -1, :]):
        raise ConstructionError("each element must lie inside a single knot span")
    cols = cols_all[:, 0, :].copy()
    if basis.closed:
        cols[cols >= basis.dim] -= basis.dim
    vals = mat.data.reshape(n_el, degree + 1, width)
    if scale_fn is not None:
        vals = vals * np.asarray(scale_fn(pts), dtype=float).reshape(n_el, degree + 1, 1)
    coeffs = np.einsum("pq,eqk->epk", vinv, vals)
    coeffs *= (half[:, None] ** -powers[None, :])[:, :, None]
    return coeffs, cols

