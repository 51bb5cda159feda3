"""O(N) host precompute feeding the GPU assembly.

Replaces the reference's O(N^2)-Python / O(N^3)-LAPACK
``build_discretization`` (assembly.py:147-172; 577 s and 34.8 GB at N=4096)
with vectorised constructions of exactly the quantities the hot path reads:

* the shared node vector (quadrature.py:87-146);
* the regular weighted rules as a BAND: row i's active nodes are the
  contiguous (seam-wrapping) node range inside supp(B_i); weights solve the
  local exactness system with the minimum-norm solution
  (quadrature.py:510-540, splines.py:491-514), batched by system shape;
* node coordinates f, speeds J (scipy BSpline, bit-identical to the
  reference's ``curve_eval`` inputs);
* the parameter-distance mode of K1 (geometry.py:127-139): a gap table of
  1/p^2 when the nodes are exactly uniform, else a per-pair formula;
* the log-part ingredients (assembly.py:206-243): per-element polynomial
  coefficients u, v, the fit normal-equation bands H and S, and for closed
  uniform simple-knot meshes the circulant inverse of H.

Nothing here is O(N^2).  The singular rules (quadrature.py:543-571) are not
built: the matrix never reads them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache
from math import comb

import numpy as np

from .errors import ConstructionError, GeometryError
from .splines import BasisSpec, active_values

DEDUP_RTOL = 1e-12        # quadrature.py:47
RANK_RTOL = 1e-10         # quadrature.py:48
EXACTNESS_TOL = 1e-11     # quadrature.py:49
DIAG_REL = 1e-7           # geometry.py:37
JFIT_DEGREE = 12          # assembly.py:82
PAIR_FAR_ORDER = 30       # quadrature.py:369
PERIODIC_CORR_ORDER = 24  # quadrature.py:53 (closed-domain weight correction)


# -- nodes ---------------------------------------------------------------------


def build_nodes(fine: BasisSpec, end_fix: bool = False) -> np.ndarray:
    """Breakpoints + midpoints, d+2 points in open end elements, extra points
    beside multiple knots, deduplicated at 1e-12 L (quadrature.py:87-146).
    The O(N^3) SVD rank check is replaced by the banded/circulant SPD check
    of the fit normal matrix (``fit_bands``).

    ``end_fix`` (opt-in deviation): the reference gives an open
    end element exactly d interior points (quadrature.py:106-108), dropping the
    m - 1 extra points its inner breakpoint of multiplicity m asks for, so a
    repeated knot next to an end element leaves the last regular rule
    rank-deficient (quadrature.py:528-531, ConstructionError).  With end_fix the
    end element keeps both: d + (m - 1) interior points."""
    d = fine.degree
    els = fine.elements
    pts = [fine.breakpoints]
    extra = fine.multiplicities - 1
    if fine.closed:
        extra = extra.copy()
        extra[0] = extra[-1] = fine.seam_multiplicity - 1
    n_inner = 1 + extra[:-1] + extra[1:]
    if not fine.closed:
        if end_fix and len(els) > 1:
            n_inner[0] = d + extra[1]
            n_inner[-1] = d + extra[-2]
        else:
            n_inner[0] = n_inner[-1] = d
    if np.all(n_inner == 1):
        mids = 0.5 * (els[:, 0] + els[:, 1])
        if fine.closed:
            pts.append(mids)
        else:
            pts.append(np.linspace(els[0, 0], els[0, 1], d + 2))
            pts.append(np.linspace(els[-1, 0], els[-1, 1], d + 2))
            if len(els) > 2:
                pts.append(mids[1:-1])
    else:
        k = n_inner.astype(int)
        e_idx = np.repeat(np.arange(len(els)), k)
        off = np.arange(k.sum()) - np.repeat(np.cumsum(k) - k, k) + 1
        lo, hi = els[e_idx, 0], els[e_idx, 1]
        pts.append(lo + (hi - lo) * (off / (k[e_idx] + 1)))
    nodes = np.sort(np.concatenate(pts))
    tol = DEDUP_RTOL * fine.length
    nodes = nodes[np.concatenate([[True], np.diff(nodes) > tol])]
    if fine.closed and fine.b - nodes[-1] <= tol:
        nodes = nodes[:-1]
    if len(nodes) < fine.dim:
        raise ConstructionError(
            f"{len(nodes)} nodes cannot satisfy Schoenberg-Whitney for {fine.dim} exactness functions")
    return nodes


# -- contiguous cyclic index ranges ----------------------------------------------


def _ranges(owner, idx, n_owner, modulus, closed):
    """For (owner, idx) incidence pairs whose per-owner index sets are
    contiguous (seam-wrapping on closed domains), return (start, length) with
    ``start`` unwrapped: it may be negative so that start..start+length-1
    runs monotonically and indices are taken modulo ``modulus``."""
    owner = np.asarray(owner, np.int64)
    idx = np.asarray(idx, np.int64)
    order = np.lexsort((idx, owner))
    owner, idx = owner[order], idx[order]
    keep = np.ones(len(idx), bool)
    keep[1:] = (owner[1:] != owner[:-1]) | (idx[1:] != idx[:-1])
    owner, idx = owner[keep], idx[keep]
    counts = np.bincount(owner, minlength=n_owner)
    if np.any(counts == 0):
        raise ConstructionError("a basis function has no support in the node/element set")
    first = np.cumsum(counts) - counts
    lo, hi = idx[first], idx[first + counts - 1]
    start = lo.copy()
    wrapped = (hi - lo + 1) != counts
    if np.any(wrapped):
        if not closed:
            raise ConstructionError("support index set is not contiguous")
        same = owner[1:] == owner[:-1]
        jump = np.flatnonzero((np.diff(idx) > 1) & same)
        jo = owner[jump]
        if len(np.unique(jo)) != len(jo) or not np.array_equal(np.sort(jo), np.flatnonzero(wrapped)):
            raise ConstructionError("support index set is not contiguous")
        s = idx[jump + 1]
        if np.any((modulus - s) + (idx[jump] + 1) != counts[jo]) or np.any(lo[jo] != 0) \
                or np.any(hi[jo] != modulus - 1):
            raise ConstructionError("support index set is not contiguous")
        # two unwrapped representations (s - modulus or s running past the
        # end); keep the one nearest the owner's position so starts stay monotone
        expect = jo * (modulus / n_owner)
        neg = s - modulus
        start[jo] = np.where(np.abs(neg - expect) <= np.abs(s - expect), neg, s)
    return start, counts


# -- regular weighted rules (quadrature.py:510-540) ---------------------------------


@dataclass
class RuleBand:
    start: np.ndarray   # (N,) int64, unwrapped first node of each rule
    width: np.ndarray   # (N,) int64
    weights: np.ndarray  # (N, WG) rule weights (zero padded)
    WG: int


def _unique_rows(key: np.ndarray):
    """(first, inv) of np.unique(key, axis=0, return_index=True, return_inverse=True) up to
    the order of the groups: rows are grouped by a 64-bit hash of their bits (a sort of n
    integers instead of a lexicographic sort of n rows), verified exactly, with the full
    row sort as the fallback on a hash collision."""
    key = np.ascontiguousarray(key, dtype=np.float64)
    bits = key.view(np.uint64)
    mult = (np.arange(1, key.shape[1] + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1)
    with np.errstate(over="ignore"):
        h = (bits * mult[None, :]).sum(axis=1, dtype=np.uint64)
    _, first, inv = np.unique(h, return_index=True, return_inverse=True)
    inv = inv.ravel()
    if not np.array_equal(bits[first][inv], bits):
        _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
        inv = inv.ravel()
    return first, inv


def regular_rule_band(parent: BasisSpec, fine: BasisSpec, nodes: np.ndarray) -> RuleBand:
    """Minimum-norm weighted rules, one per parent function, exact on every
    fine function overlapping its support (quadrature.py:510-540).

    Active nodes = nodes where B_i != 0 (quadrature.py:525); exactness
    functions = fine functions active on the fine elements of supp(B_i)
    (splines.py:374-382); moments mu_j = int B_i Bbar_j by per-element
    Gauss of order (p+d)//2+2 (splines.py:491-514).  The local systems are
    solved batched (SVD pseudo-inverse = minimum-norm solution for the
    full-row-rank systems the reference accepts).
    """
    nq = len(nodes)
    N, NE = parent.dim, fine.dim
    p, d = parent.degree, fine.degree
    closed = fine.closed

    # active nodes per parent function
    pv, pc = active_values(parent, nodes)
    nz = pv != 0.0
    q_of = np.broadcast_to(np.arange(nq)[:, None], pv.shape)[nz]
    n_start, n_len = _ranges(pc[nz], q_of, N, nq, closed)

    # per fine element: Gauss moments E_e[a, b] = int_e Bc_a Bf_b
    els = fine.elements
    ne = len(els)
    order = (p + d) // 2 + 2
    xg, wg = np.polynomial.legendre.leggauss(order)
    half = 0.5 * (els[:, 1] - els[:, 0])
    mid = 0.5 * (els[:, 0] + els[:, 1])
    gp = (mid[:, None] + half[:, None] * xg[None, :]).ravel()
    cv, cc = active_values(parent, gp)
    fv, fc = active_values(fine, gp)
    cv = cv.reshape(ne, order, p + 1)
    fv = fv.reshape(ne, order, d + 1)
    cc = cc.reshape(ne, order, p + 1)[:, 0, :]
    fc = fc.reshape(ne, order, d + 1)[:, 0, :]
    E = np.einsum("eg,ega,egb->eab", half[:, None] * wg[None, :], cv, fv)

    # elements of supp(B_i): fine elements where i is active
    e_of = np.broadcast_to(np.arange(ne)[:, None], cc.shape).ravel()
    e_start, e_len = _ranges(cc.ravel(), e_of, N, ne, closed)
    WE = int(e_len.max())
    eidx = (e_start[:, None] + np.arange(WE)[None, :])
    emask = np.arange(WE)[None, :] < e_len[:, None]
    eidx = np.mod(eidx, ne)

    # exactness functions: union of fine active functions over those elements
    fcu = fc[eidx]  # (N, WE, d+1)
    fcu_unw = fcu.astype(np.int64).copy()
    if closed:
        # unwrap relative to the first element's first function
        ref = fcu[:, :1, :1]
        fcu_unw = ref + np.mod(fcu - ref + NE // 2, NE) - NE // 2
    big = np.iinfo(np.int64).max // 4
    jlo = np.where(emask[:, :, None], fcu_unw, big).min(axis=(1, 2))
    jhi = np.where(emask[:, :, None], fcu_unw, -big).max(axis=(1, 2))
    j_len = jhi - jlo + 1
    WJ = int(j_len.max())
    jidx_unw = jlo[:, None] + np.arange(WJ)[None, :]
    jmask = np.arange(WJ)[None, :] < j_len[:, None]
    jidx = np.mod(jidx_unw, NE)

    # mu[i, r] = sum_e sum_{a: cc=i} sum_{b: fc=jsel_r} E_e[a, b]
    ccu = cc[eidx]  # (N, WE, p+1)
    amask = (ccu == np.arange(N)[:, None, None]) & emask[:, :, None]
    Ee = E[eidx]  # (N, WE, p+1, d+1)
    rowE = np.einsum("nwa,nwab->nwb", amask.astype(float), Ee)  # (N, WE, d+1)
    match = (fcu[:, :, :, None] == jidx[:, None, None, :]) & jmask[:, None, None, :]
    mu = np.einsum("nwb,nwbr->nr", rowE, match.astype(float))

    # local collocation matrices: Bbar_{jsel_r}(eta_{nsel_c})
    WN = int(n_len.max())
    nidx = np.mod(n_start[:, None] + np.arange(WN)[None, :], nq)
    nmask = np.arange(WN)[None, :] < n_len[:, None]
    fvn, fcn = active_values(fine, nodes)
    fvg, fcg = fvn[nidx], fcn[nidx]  # (N, WN, d+1)
    eq = (fcg[:, None, :, :] == jidx[:, :, None, None])  # (N, WJ, WN, d+1)
    local = np.einsum("njcb,ncb->njc", eq.astype(float), fvg)
    local *= jmask[:, :, None] & nmask[:, None, :]

    weights = np.zeros((N, WN))
    shapes = np.stack([j_len, n_len], axis=1)
    for sj, sn in np.unique(shapes, axis=0):
        sel = np.flatnonzero((j_len == sj) & (n_len == sn))
        Am = local[sel][:, :sj, :sn]
        bm = mu[sel][:, :sj]
        if sj > sn:   # more exactness functions than nodes: rank < len(jsel) (quadrature.py:528-531)
            # padded / seam-wrapped ranges hold zero or repeated rows: count
            # the distinct live exactness functions
            lm = (Am != 0.0).any(axis=2) | (bm != 0.0)
            for k in range(len(sel)):
                if len(np.unique(jidx[sel[k], :sj][lm[k]])) > sn:
                    raise ConstructionError(
                        f"rank-deficient local collocation matrix for weight {int(sel[k])}")
        # identical local systems (every rule of a uniform mesh, up to the ends) are solved
        # once: the same inputs give the same bits
        key = np.concatenate([Am.reshape(len(sel), -1), bm], axis=1)
        first, inv = _unique_rows(key)
        Am, bm = Am[first], bm[first]
        u_, s_, vt = np.linalg.svd(Am, full_matrices=False)
        if np.any(s_[:, -1] <= max(sj, sn) * np.finfo(float).eps * s_[:, 0]):
            raise ConstructionError("rank-deficient local collocation matrix for a weight")
        w = np.einsum("kij,ki->kj", vt, np.einsum("kji,kj->ki", u_, bm) / s_)
        resid = np.linalg.norm(np.einsum("kjc,kc->kj", Am, w) - bm, axis=1)
        if np.any(resid > EXACTNESS_TOL):
            raise ConstructionError(f"regular rule exactness residual {resid.max():.2e}")
        weights[sel, :sn] = w[inv.ravel()]
    return RuleBand(start=n_start, width=n_len, weights=weights, WG=WN)


# -- geometry at the nodes + K1 parameter-distance mode ------------------------------


K1_MODE_TABLE = 0        # 1/p^2 gap table (exactly uniform nodes)
K1_MODE_OPEN = 1         # p = |t - s|
K1_MODE_CLOSED = 2       # p = (L/pi)|sin(pi |t - s| / L)|, unwrapped |t - s|


def uniform_spacing(nodes: np.ndarray):
    """Spacing if the nodes are a + k*Delta EXACTLY with Delta a power of two
    (then every |eta_r - eta_q| equals |r - q|*Delta bit for bit)."""
    if len(nodes) < 2:
        return None
    delta = nodes[1] - nodes[0]
    if delta <= 0 or np.frexp(delta)[0] != 0.5:
        return None
    ref = nodes[0] + np.arange(len(nodes)) * delta
    return float(delta) if np.array_equal(ref, nodes) else None


def k1_distance_table(nodes, closed, length):
    """1/p^2 per node-index gap, p computed exactly as the reference does
    (geometry.py:134-139) from the unwrapped |t - s|."""
    delta = uniform_spacing(nodes)
    if delta is None:
        return None
    x = np.abs(nodes - nodes[0])
    if closed:
        p = (length / np.pi) * np.abs(np.sin(np.pi * x / length))
    else:
        p = x
    with np.errstate(divide="ignore"):
        inv = 1.0 / (p * p)
    inv[0] = 0.0
    return inv


def near_diagonal_pairs(nodes, closed, a, length, speed):
    """Distinct node pairs within eps_diag = DIAG_REL L of each other take the
    continuity limit J(mid)^2 (geometry.py:237-245) instead of the divided
    difference.  Returns (K, table) with table[q, k-1] = J(mid)^2 for the pair
    (q, q+k mod nq) when near, else 0; K = 0 (table None) when no distinct
    pair is near (uniform meshes).  ``speed`` evaluates J at parameters; a is
    the start of the curve's parameter domain."""
    eps = DIAG_REL * length
    nq = len(nodes)
    K = 0
    while K + 1 < nq:
        j = np.arange(nq) + K + 1
        if not closed:
            j = j[j < nq]
        delta = nodes[np.mod(j, nq)] - nodes[: len(j)]
        if closed:
            delta = delta - length * np.round(delta / length)
        if not np.any(np.abs(delta) <= eps):
            break
        K += 1
    if K == 0:
        return 0, None
    table = np.zeros((nq, K))
    for k in range(1, K + 1):
        q = np.arange(nq if closed else nq - k)
        s = nodes[q]
        delta = nodes[np.mod(q + k, nq)] - s
        if closed:
            delta = delta - length * np.round(delta / length)
        near = np.abs(delta) <= eps
        if near.any():
            mid = s[near] + 0.5 * delta[near]
            if closed:
                mid = a + np.mod(mid - a, length)
            table[q[near], k - 1] = speed(mid) ** 2
    return K, table


# -- pair log moments: the analytic near-gap table (quadrature.py:182-197,372-410) ----


def _log_power_bracket(j, z1, z2):
    """[z^{j+1}/(j+1) (ln|z| - 1/(j+1))] between z1 and z2 with the removable
    limit at z = 0 (quadrature.py:182-197)."""
    def F(z):
        z = np.asarray(z, float)
        out = np.zeros_like(z)
        nz = z != 0.0
        zz = z[nz]
        out[nz] = zz ** (j + 1) / (j + 1) * (np.log(np.abs(zz)) - 1.0 / (j + 1))
        return out
    return F(z2) - F(z1)


def near_moments_closed_form(da, db, he, hf, delta):
    """Exact centred double log moments M[k,a,b] = int int u^a v^b
    ln|v - u - delta| over (-he/2,he/2) x (-hf/2,hf/2) (quadrature.py:372-410),
    same operation order as the reference (its round-off is part of the
    reference result at high powers)."""
    he, hf, delta = np.broadcast_arrays(np.asarray(he, float), np.asarray(hf, float),
                                        np.asarray(delta, float))
    n = he.shape[0]
    out = np.zeros((n, da + 1, db + 1))
    pmax = da + db + 1
    for sgn in (1.0, -1.0):
        xi = sgn * 0.5 * hf
        z1 = xi - delta - 0.5 * he
        z2 = xi - delta + 0.5 * he
        llog = [_log_power_bracket(p, z1, z2) for p in range(pmax + 1)]
        lpow = [(z2 ** (p + 1) - z1 ** (p + 1)) / (p + 1) for p in range(pmax + 1)]
        for b in range(db + 1):
            for m in range(b + 1):
                cm = sgn * comb(b, m) / (m + 1)
                for a in range(da + 1):
                    acc = np.zeros(n)
                    for r in range(a + 1):
                        for q in range(b - m + 1):
                            p = r + q + m + 1
                            coef = (cm * comb(a, r) * comb(b - m, q) * (-1.0) ** (r + q)
                                    * (xi - delta) ** (a - r) * xi ** (b - m - q))
                            acc += coef * (llog[p] - lpow[p] / (m + 1))
                    out[:, a, b] += acc
    return out


@lru_cache(maxsize=16)
def unit_near_table(da: int, db: int):
    """Unit-width closed-form moments for integer gaps -1, 0, +1 (rows ordered
    by keff = -1, 0, 1; delta = -keff), cached like the reference's stack."""
    keff = np.array([-1.0, 0.0, 1.0])
    t = near_moments_closed_form(da, db, np.ones(3), np.ones(3), -keff)
    t.setflags(write=False)
    return t


@lru_cache(maxsize=8)
def gauss_unit(order: int):
    """Gauss-Legendre nodes/weights on (-0.5, 0.5) (quadrature.py:56-71)."""
    x, w = np.polynomial.legendre.leggauss(order)
    return 0.5 * x, 0.5 * w


def centred_monomial_integrals(n: int):
    """c_p = int_{-1/2}^{1/2} u^p du (quadrature.py:497-498)."""
    pa = np.arange(n + 1)
    return np.where(pa % 2 == 0, 0.5 ** pa / (pa + 1.0), 0.0)


def uniform_width(fine: BasisSpec):
    widths = fine.elements[:, 1] - fine.elements[:, 0]
    h = widths.mean()
    if not np.allclose(widths, h, rtol=DEDUP_RTOL):
        raise ConstructionError("pair log moments require a uniform element mesh")
    return float(h)


def is_uniform_mesh(fine: BasisSpec) -> bool:
    widths = fine.elements[:, 1] - fine.elements[:, 0]
    return bool(np.allclose(widths, widths.mean(), rtol=DEDUP_RTOL))


# touching / overlapping element pairs (separation <= this fraction of the
# larger width) use the closed form, as the reference's |gap| <= 1 entries
# (quadrature.py:458); every other pair is analytic and takes Gauss
NEAR_TOUCH = 1e-9
# far-pair Gauss orders by separation (< 2, < 8, >= 8 larger widths); must match
# the tier sizes compiled into wq_general.cu
GEN_GAUSS_TIERS = (30, 16, 12)


def log_gauss_unit(n: int, levels: int = 30, ratio: float = 0.25, m: int = 20):
    """n-point Gauss rule for the weight -ln x on (0, 1): Stieltjes procedure
    on a discrete measure (composite Gauss-Legendre on panels graded toward
    0), eigen-decomposition of the Jacobi matrix.  Exact to ~1e-16 for
    polynomials of degree <= 2n - 1 (tests/test_host.py)."""
    x, w = np.polynomial.legendre.leggauss(m)
    edges = np.concatenate([[0.0], ratio ** np.arange(levels, -1, -1.0)])
    lo, hi = edges[:-1, None], edges[1:, None]
    X = (0.5 * (lo + hi) + 0.5 * (hi - lo) * x).ravel()
    Wt = (0.5 * (hi - lo) * w).ravel() * (-np.log(X))
    a = np.zeros(n)
    b = np.zeros(n)
    p_prev, p = np.zeros_like(X), np.ones_like(X)
    nrm_prev = 1.0
    for k in range(n):
        nrm = np.sum(Wt * p * p)
        a[k] = np.sum(Wt * X * p * p) / nrm
        b[k] = nrm / nrm_prev if k else 0.0
        p_prev, p, nrm_prev = p, (X - a[k]) * p - b[k] * p_prev, nrm
    jac = np.diag(a) + np.diag(np.sqrt(b[1:]), 1) + np.diag(np.sqrt(b[1:]), -1)
    ev, vec = np.linalg.eigh(jac)
    return ev, Wt.sum() * vec[0] ** 2


# touching pairs of unequal widths: Duffy split of the pair rectangle at the
# shared corner -> ln(xi) (log-weighted rule) + smooth terms (Gauss-Legendre);
# sizes compiled into wq_general.cu
TOUCH_XI, TOUCH_ETA, TOUCH_LOG = 16, 30, 14
TOUCH_MAX_RATIO = 8.0


def touch_rules() -> np.ndarray:
    """Packed [x16, w16, x30, w30 (Gauss-Legendre on (0,1)), xl14, wl14
    (weight -ln x on (0,1))]."""
    out = []
    for n in (TOUCH_XI, TOUCH_ETA):
        x, w = np.polynomial.legendre.leggauss(n)
        out += [0.5 * (x + 1.0), 0.5 * w]
    out += list(log_gauss_unit(TOUCH_LOG))
    return np.concatenate(out)


def element_pair_geometry(fine: BasisSpec):
    """Widths, midpoints and, per outer element e, the contiguous (cyclic on
    closed meshes) range of inner elements f whose separation is at most
    NEAR_TOUCH x max(h_e, h_f): f = lo[e] + k (mod n), k < cnt[e].
    Same predicate and operation order as the restated reference recipe."""
    els = fine.elements
    n = len(els)
    h = els[:, 1] - els[:, 0]
    mid = 0.5 * (els[:, 0] + els[:, 1])
    L = fine.length
    win = 4
    while True:
        win = min(win, n // 2 if fine.closed else n - 1)
        off = np.arange(-win, win + 1)
        f = np.arange(n)[:, None] + off[None, :]
        valid = np.ones_like(f, bool) if fine.closed else (f >= 0) & (f < n)
        f = np.mod(f, n)
        delta = mid[:, None] - mid[f]
        if fine.closed:
            delta = delta - L * np.round(delta / L)
        sep = np.abs(delta) - 0.5 * (h[:, None] + h[f])
        near = valid & (sep <= NEAR_TOUCH * np.maximum(h[:, None], h[f]))
        edge = near[:, 0] | near[:, -1]
        full = (2 * win + 1 >= n) if fine.closed else (win >= n - 1)
        if not edge.any() or full:
            break
        win *= 2
    if fine.closed and 2 * win + 1 > n:  # each residue once
        near, off = near[:, :n], off[:n]
    first = np.argmax(near, axis=1)
    last = near.shape[1] - 1 - np.argmax(near[:, ::-1], axis=1)
    lo = np.mod(np.arange(n) + off[first], n)
    cnt = last - first + 1   # gaps inside the range also take the near route
    # touching pairs of unequal widths: the Duffy rules are sized for ratios <= 8
    f = np.mod(np.arange(n)[:, None] + off[None, :], n)
    ratio = np.where(near, h[f] / h[:, None], 1.0)
    ratio = np.maximum(ratio, 1.0 / ratio)
    if ratio.max() > TOUCH_MAX_RATIO:
        raise ConstructionError(
            f"adjacent element width ratio {ratio.max():.3g} > {TOUCH_MAX_RATIO:g} unsupported")
    return h, mid, lo.astype(np.int64), cnt.astype(np.int64)


# -- fit normal equations (assembly.py:233-243 -> banded) -------------------


def fit_bands(fine: BasisSpec, parent: BasisSpec, nodes, J):
    """H = Bt^T Bt (N_E x N_E, half-bandwidth d, seam-cyclic on closed meshes)
    and S = Bt^T (J Bpar^T) (N_E x N) as sparse matrices, with Bt the fine
    basis at the nodes.  C = H^{-1} S is the reference's QR fit
    (assembly.py:237-243) through its normal equations (<= 4e-15)."""
    import scipy.sparse as sp

    nq = len(nodes)
    fv, fc = active_values(fine, nodes)
    pv, pc = active_values(parent, nodes)
    rows = np.repeat(np.arange(nq), fv.shape[1])
    Bt = sp.csr_matrix((fv.ravel(), (rows, fc.ravel())), shape=(nq, fine.dim))
    rows = np.repeat(np.arange(nq), pv.shape[1])
    Bp = sp.csr_matrix(((pv * J[:, None]).ravel(), (rows, pc.ravel())), shape=(nq, parent.dim))
    H = (Bt.T @ Bt).tocsr()
    S = (Bt.T @ Bp).tocsc()
    return H, S


def band_of_columns(S, closed):
    """Column band of a sparse matrix: per column j the unwrapped start row and
    a dense zero-padded (ncols, W) block with vals[j, k] = S[start_j + k, j]."""
    S = S.tocsc()
    S.sort_indices()
    nr, ncol = S.shape
    col_of = np.repeat(np.arange(ncol), np.diff(S.indptr))
    start, length = _ranges(col_of, S.indices, ncol, nr, closed)
    W = int(length.max())
    vals = np.zeros((ncol, W))
    pos = np.mod(S.indices - start[col_of], nr)
    vals[col_of, pos] = S.data
    return start, vals


def circulant_inverse(H, nfine):
    """First row of H^{-1} for a circulant SPD H (closed uniform simple knots).

    Returns (hinv, K): |H^{-1}[0, k]| < 1e-18 |H^{-1}[0, 0]| for K < |k| <= n/2.
    For n <= 512 the exact symbol inverse (FFT) is returned with K = n // 2.
    For larger n the taps decay geometrically and are computed entrywise
    accurately from the bi-infinite banded Toeplitz inverse (banded Cholesky
    solve of a centred segment), avoiding the ~1e-15 relative noise floor an
    FFT leaves on the tail; periodisation corrections are below 1e-18 for
    n > 2K.
    """
    import scipy.linalg

    row = np.asarray(H[0].todense()).ravel()
    lam = np.real(np.fft.fft(row))
    if lam.min() <= 0 or lam.min() <= RANK_RTOL ** 2 * lam.max():
        raise ConstructionError("node vector does not resolve the refined space")
    if nfine <= 512:
        return np.real(np.fft.ifft(1.0 / lam)), nfine // 2
    # symmetric band t_0..t_b of the Toeplitz symbol
    b = 0
    for k in range(1, nfine // 2):
        if row[k] != 0.0 or row[nfine - k] != 0.0:
            b = k
    t = 0.5 * (row[: b + 1] + np.concatenate([[row[0]], row[nfine - np.arange(1, b + 1)]]))
    M = min(nfine // 2 - 1, 800)
    size = 2 * M + 1
    ab = np.zeros((b + 1, size))
    for k in range(b + 1):
        ab[k, : size - k] = t[k]
    rhs = np.zeros(size)
    rhs[M] = 1.0
    x = scipy.linalg.solveh_banded(ab, rhs, lower=True)
    taps = x[M:]                      # H^{-1}[0, k], k = 0..M
    small = np.flatnonzero(np.abs(taps) < 1e-18 * abs(taps[0]))
    K = int(small[0]) if len(small) else M
    if 2 * K + 1 >= nfine:
        return np.real(np.fft.ifft(1.0 / lam)), nfine // 2
    hinv = np.zeros(nfine)
    hinv[: K + 1] = taps[: K + 1]
    hinv[nfine - K:] = taps[1: K + 1][::-1]
    return hinv, K


def fit_cholesky(H, bw: int, closed: bool):
    """Cholesky factor of the fit normal matrix H (N_E x N_E, half-bandwidth
    bw).  Open meshes: plain banded factor.  Closed meshes: H couples across
    the seam, so the factor is arrow-shaped: the leading m = N_E - bw block is
    banded (Lb), the last bw rows are dense (L21 = A21 L11^{-T}) plus a small
    dense Schur factor L22.  Returns (Lb, bw, L21, L22) with Lb[k, j] = L[k, k-j].
    Raises ConstructionError when H is not numerically SPD (the reference's
    rank check, assembly.py:238-242 / quadrature.py:136-140)."""
    import scipy.linalg

    H = H.tocsr()
    n = H.shape[0]
    m = n - bw if closed else n
    if closed and m <= bw:
        raise ConstructionError("closed mesh too small for the cyclic banded fit")
    ab = np.zeros((bw + 1, m))
    for j in range(bw + 1):
        ab[j, : m - j] = H[:m, :m].diagonal(-j)
    try:
        lo = scipy.linalg.cholesky_banded(ab, lower=True)
    except np.linalg.LinAlgError as exc:
        raise ConstructionError("node vector does not resolve the refined space") from exc
    Lb = np.zeros((m, bw + 1))
    for j in range(bw + 1):
        Lb[j:, j] = lo[j, : m - j]
    L21 = L22 = None
    diag = lo[0]
    if closed:
        A21 = H[m:, :m].toarray()
        L21 = scipy.linalg.solve_banded((bw, 0), lo, A21.T).T
        Sch = H[m:, m:].toarray() - L21 @ L21.T
        try:
            L22 = np.linalg.cholesky(Sch)
        except np.linalg.LinAlgError as exc:
            raise ConstructionError("node vector does not resolve the refined space") from exc
        diag = np.concatenate([diag, np.diag(L22)])
        L21 = np.ascontiguousarray(L21)
        L22 = np.ascontiguousarray(L22)
    if diag.min() ** 2 <= RANK_RTOL ** 2 * diag.max() ** 2:
        raise ConstructionError("node vector does not resolve the refined space")
    return Lb, bw, L21, L22


def inverse_decay_rows(Lb: np.ndarray, bw: int, tol: float = 1e-20, probes: int = 9,
                       window: int = 2048) -> int:
    """Rows after which a column of L^{-1} and of L^{-T} (L the banded factor,
    Lb[k, j] = L[k, k-j]) has fallen below ``tol`` of its peak, maximised over
    unit-vector probes spread along the band (forward and backward); -1 when a
    probe does not decay within ``window`` rows.  Sizes the warm-up of the
    segmented device solves (wq_band_solve_seg)."""
    import scipy.linalg
    m = Lb.shape[0]
    lo = np.zeros((bw + 1, m))
    for j in range(bw + 1):
        lo[j, : m - j] = Lb[j:, j]
    worst = 0
    for k in np.unique(np.linspace(0, m - 1, probes).astype(int)):
        # (probes near the ends see fewer rows; the interior ones bound the decay)
        for fwd in (True, False):
            n = min(window, m - k) if fwd else min(window, k + 1)
            if n < 2:
                continue
            e = np.zeros(n)
            if fwd:       # L x = e_k restricted to rows k .. k + n - 1 (the same decay)
                sub = lo[:, k:k + n].copy()
                e[0] = 1.0
                x = np.abs(scipy.linalg.solve_banded((bw, 0), sub, e))
            else:         # L^T x = e_k on rows k - n + 1 .. k, read backwards
                sub = np.zeros((bw + 1, n))
                for j in range(bw + 1):   # upper band of L^T: row r, column r + j holds L[r + j, r]
                    sub[bw - j, j:] = lo[j, k - n + 1: k + 1 - j]
                e[-1] = 1.0
                x = np.abs(scipy.linalg.solve_banded((0, bw), sub, e))[::-1]
            last = int(np.flatnonzero(x >= tol * x.max())[-1])   # last entry still above tol
            if last >= n - 1:
                if n == window:
                    return -1          # no decay within the window
                continue               # cut short by the end of the band: no information
            worst = max(worst, last + 1)
    return worst
