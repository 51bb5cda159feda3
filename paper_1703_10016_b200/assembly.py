"""Drop-in Galerkin assembly entry points (mirrors wqbem/assembly.py).

Same names, arguments, return types and error behaviour as the reference:

    build_discretization(curve, space, nref) -> Discretization   (assembly.py:147)
    assemble_ik1(disc) -> ndarray[N, N]                           (assembly.py:175)
    assemble_ik2(disc) -> ndarray[N, N]                           (assembly.py:186)
    assemble_weighted_matrix(disc) -> (M, {"kernel_evals"}, s)    (assembly.py:248)
    scale_and_symmetrize(M) -> (A, defect)                        (assembly.py:262)
    assemble_b1_weighted(disc, dirichlet) -> ndarray[N]           (assembly.py:312)
    assemble_b1(curve, space, dirichlet, order=16)                (assembly.py:287)

The O(N^2) work runs ONLY on the GPU through the C-ABI library (``_lib``);
there is no CPU fallback -- without the library or a CUDA device these raise
``DeviceError``.  ``build_discretization`` is an O(N) host precompute (see
``precompute``); the O(N^3) singular rules the matrix never reads are not
built.

Formulation.  With C = H^{-1} S the node least-squares fit
(assembly.py:233-243), Theta and D the element-pair log moments,

    X  = IK1 + X2,     X2 = (2 Theta - C^T D) C,
    M  = (X + X^T)/2 = sym(IK1 + IK2),     A = -(X + X^T) / (4 pi).

``assemble_weighted_matrix`` returns the symmetric M (it differs from the
reference's unsymmetrised M only by the reference's own pre-symmetrisation
defect, <= 2.5e-14 relative), so ``scale_and_symmetrize`` of it is exact.
Device-resident variants (``assemble_matrix_device``) return torch tensors.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import precompute as PC
from .errors import ConstructionError, DeviceError, GeometryError, UsageError
from .geometry import BoundaryCurve, as_curve, parametric_speed
from .splines import BasisSpec, RefinedBasis, active_values, as_basis, local_basis_coeffs, refine_uniform

__all__ = [
    "NodeVector",
    "WeightedRule",
    "Discretization",
    "build_discretization",
    "assemble_ik1",
    "assemble_ik2",
    "assemble_weighted_matrix",
    "assemble_matrix_device",
    "scale_and_symmetrize",
    "assemble_b1_weighted",
    "assemble_b1",
    "assemble_b2",
    "basis_values",
]

TWO_PI = 2.0 * np.pi
_GRADE_LEVELS = 14
_GRADE_RATIO = 0.3


def _check_space(curve: BoundaryCurve, space: BasisSpec):
    gb = curve.basis
    if space.closed != gb.closed:
        raise UsageError("solution space and curve disagree on closedness")
    if abs(space.a - gb.a) > 1e-12 or abs(space.b - gb.b) > 1e-12:
        raise UsageError("solution space and curve have different domains")


def basis_values(basis, pts) -> np.ndarray:
    """Dense (n_pts, dim) matrix of basis values (assembly.py:101-108)."""
    basis = as_basis(basis)
    vals, cols = active_values(basis, basis._check_domain(pts))
    out = np.zeros((len(vals), basis.dim))
    np.add.at(out, (np.repeat(np.arange(len(vals)), vals.shape[1]), cols.ravel()), vals.ravel())
    return out


@dataclass(frozen=True)
class NodeVector:
    """Shared quadrature nodes (quadrature.py:74-84)."""

    nodes: np.ndarray
    refined: RefinedBasis = field(repr=False)
    element_index: np.ndarray = field(repr=False)

    @property
    def n(self) -> int:
        return len(self.nodes)


@dataclass
class LogPart:
    """Host-side ingredients of the log part (assembly.py:206-243)."""

    path: str                      # "circulant" | "general"
    h: float
    da: int                        # P = p + JFIT_DEGREE
    db: int                        # refined degree d
    n_el: int
    near_unit: np.ndarray          # (3, da+1, db+1)
    s_start: np.ndarray            # (N,) S column band
    s_w: np.ndarray                # (N, ws)
    # circulant
    e_start: np.ndarray = None
    U: np.ndarray = None           # (N, tu, da+1)
    v0: np.ndarray = None          # (db+1, db+1)
    hinv_taps: np.ndarray = None   # (2K+1,)
    uext: np.ndarray = None        # (N, ktot) [2U | -S_i | 0] for the DMMA kernel
    s_span: int = None             # fit rows under the S bands of 64 columns (lazy)
    nApad: int = 0
    zstride: int = 0
    # general
    u: np.ndarray = None
    v: np.ndarray = None
    u_el: np.ndarray = None
    u_loc: np.ndarray = None
    v_el: np.ndarray = None
    v_loc: np.ndarray = None
    Lb: np.ndarray = None          # banded Cholesky factor of H (leading block if cyclic)
    bw: int = 0
    L21: np.ndarray = None         # cyclic meshes: seam coupling rows of the arrow factor
    L22: np.ndarray = None
    # graded (non-uniform) meshes: per-pair blocks instead of the gap table
    graded: bool = False
    elh: np.ndarray = None         # (n_el,) widths
    elm: np.ndarray = None         # (n_el,) midpoints
    near_lo: np.ndarray = None     # (n_el,) first near inner element (cyclic)
    near_cnt: np.ndarray = None    # (n_el,) number of near inner elements
    ucols: np.ndarray = None
    vcols: np.ndarray = None
    seg_k0: int = None             # warm-up rows of the segmented H^{-1} solves


@dataclass(frozen=True)
class WeightedRule:
    """One regular weighted rule on the shared node vector (quadrature.py:150-168):
    tag ("basis", i), active node indices, weights."""

    tag: tuple
    idx: np.ndarray
    weights: np.ndarray

    def apply(self, values_at_nodes) -> float:
        return float(self.weights @ np.asarray(values_at_nodes)[self.idx])

    def full_weights(self, n_quad: int) -> np.ndarray:
        w = np.zeros(n_quad)
        w[self.idx] = self.weights
        return w


@dataclass
class Discretization:
    """Solution space, shared node vector and the banded regular rules
    (mirrors assembly.py:131-144; G and Bpar are exposed lazily as dense
    arrays for compatibility, the GPU reads the band)."""

    curve: BoundaryCurve
    space: BasisSpec
    refined: RefinedBasis
    nodes: NodeVector
    rules: PC.RuleBand
    J_nodes: np.ndarray = field(repr=False)
    f_nodes: np.ndarray = field(repr=False)
    k1_mode: int = 0
    invp2: np.ndarray = field(default=None, repr=False)
    near_k: int = 0                # distinct node pairs within eps_diag (geometry.py:237-245)
    near_j2: np.ndarray = field(default=None, repr=False)
    rule_seconds: float = 0.0
    _logpart: object = field(default=None, repr=False)
    _dev: dict = field(default_factory=dict, repr=False)

    @property
    def regular_rules(self) -> list:
        """The regular rules as the reference's list of WeightedRule
        (assembly.py:139, quadrature.py:510-540), built from the band on first
        use; the device path reads the band (``rules``)."""
        if "regular_rules" not in self._dev:
            rb, nq = self.rules, self.nodes.n
            out = []
            for i in range(len(rb.start)):
                w = int(rb.width[i])
                idx = np.mod(rb.start[i] + np.arange(w), nq)
                order = np.argsort(idx, kind="stable")
                out.append(WeightedRule(("basis", i), idx[order], rb.weights[i, :w][order].copy()))
            self._dev["regular_rules"] = out
        return self._dev["regular_rules"]

    @property
    def singular_rules(self):
        """The singular (log) rules of Alg. 2 are not built: the matrix never
        reads them and the reference builds them in O(N^3) time /
        O(N^2) memory (quadrature.py:543-571).  Raises UsageError, so the
        reference's ``--dump-rules`` path fails with a clear message."""
        raise UsageError("singular rules are not built by the B200 backend (unused by the "
                         "matrix, SURVEY F3); dump them with the reference's build_singular_rules")

    @property
    def G(self) -> np.ndarray:
        """Dense (dim, n_quad) rule weights times J (assembly.py:160)."""
        N, nq = self.space.dim, self.nodes.n
        g = np.zeros((N, nq))
        rb = self.rules
        for w in range(rb.WG):
            m = w < rb.width
            q = np.mod(rb.start[m] + w, nq)
            g[np.flatnonzero(m), q] += rb.weights[m, w] * self.J_nodes[q]
        return g

    @property
    def Bpar(self) -> np.ndarray:
        return basis_values(self.space, self.nodes.nodes).T

    @property
    def closed(self) -> bool:
        return self.space.closed


def build_discretization(curve, space, nref: int, *, end_node_fix: bool = False) -> Discretization:
    """Refine, build nodes and the banded regular rules, and sample the curve
    at the nodes (assembly.py:147-172), in O(N) host time.

    ``end_node_fix`` (keyword-only, opt-in deviation from the reference): keep
    the extra nodes a repeated knot next to an open end element asks for, which
    the reference drops (quadrature.py:106-108) and then fails on with a
    rank-deficient last rule (ConstructionError, quadrature.py:528-531); see
    ``precompute.build_nodes``."""
    curve = as_curve(curve)
    space = as_basis(space)
    _check_space(curve, space)
    t0 = time.perf_counter()
    refined = refine_uniform(space, nref)
    fine = refined.basis
    nodes = PC.build_nodes(fine, end_fix=end_node_fix)
    rules = PC.regular_rule_band(space, fine, nodes)
    rule_seconds = time.perf_counter() - t0
    b = curve.basis
    f_nodes = curve.spline(0)(np.clip(nodes, b.a, b.b))
    J = parametric_speed(curve, nodes)
    near_k, near_j2 = PC.near_diagonal_pairs(nodes, space.closed, b.a, curve.length,
                                             lambda s: parametric_speed(curve, s))
    invp2 = PC.k1_distance_table(nodes, space.closed, curve.length) if near_k == 0 else None
    if invp2 is not None:
        mode = _lib.WQ_K1_TABLE
    else:
        mode = _lib.WQ_K1_CLOSED if space.closed else _lib.WQ_K1_OPEN
    el_idx = np.clip(np.searchsorted(fine.breakpoints, nodes, side="right") - 1, 0,
                     fine.n_elements - 1)
    return Discretization(curve=curve, space=space, refined=refined,
                          nodes=NodeVector(nodes=nodes, refined=refined, element_index=el_idx),
                          rules=rules, J_nodes=J, f_nodes=f_nodes, k1_mode=mode, invp2=invp2,
                          near_k=near_k, near_j2=near_j2, rule_seconds=rule_seconds)


# -- log-part host ingredients ---------------------------------------------------------


def _incidence(cols, n_fun):
    """(element, local) incidences of every function, padded with -1."""
    n_el, w = cols.shape
    fun = cols.ravel()
    el = np.repeat(np.arange(n_el), w)
    loc = np.tile(np.arange(w), n_el)
    order = np.lexsort((el, fun))
    fun, el, loc = fun[order], el[order], loc[order]
    counts = np.bincount(fun, minlength=n_fun)
    width = int(counts.max())
    first = np.cumsum(counts) - counts
    slot = np.arange(len(fun)) - first[fun]
    E = np.full((n_fun, width), -1, np.int64)
    L = np.zeros((n_fun, width), np.int64)
    E[fun, slot] = el
    L[fun, slot] = loc
    return E, L, counts


def _is_circulant(disc: Discretization) -> bool:
    fine = disc.refined.basis
    return (fine.closed and disc.refined.nref == 1 and np.all(fine.multiplicities == 1)
            and fine.seam_multiplicity == 1 and fine.dim == fine.n_elements)


# route uniform meshes through the per-pair (graded-mesh) kernels too; tests use
# it to pin those kernels against the reference's uniform-mesh outputs
_FORCE_PER_PAIR = False


def _log_part(disc: Discretization) -> LogPart:
    if disc._logpart is not None:
        return disc._logpart
    fine, space = disc.refined.basis, disc.space
    # the reference raises ConstructionError on graded meshes (quadrature.py:489-491);
    # here they take the per-pair route
    graded = _FORCE_PER_PAIR or not PC.is_uniform_mesh(fine)
    h = None if graded else PC.uniform_width(fine)
    d = fine.degree
    da = space.degree + PC.JFIT_DEGREE
    curve = disc.curve
    cb = curve.basis

    def jac(pts):
        return np.linalg.norm(curve.spline(1)(np.clip(pts, cb.a, cb.b)), axis=-1)

    u, ucols = local_basis_coeffs(space, fine.elements, da, scale_fn=jac)
    v, vcols = local_basis_coeffs(fine, fine.elements, d)
    H, S = PC.fit_bands(fine, space, disc.nodes.nodes, disc.J_nodes)
    s_start, s_w = PC.band_of_columns(S, fine.closed)
    lp = LogPart(path="general", h=h, da=da, db=d, n_el=fine.n_elements,
                 near_unit=np.ascontiguousarray(PC.unit_near_table(da, d)),
                 s_start=s_start, s_w=s_w)
    N = space.dim
    if not graded and _is_circulant(disc):
        n = fine.n_elements
        _, _, counts = _incidence(ucols, N)
        tu = int(counts.max())
        # with simple knots supp(B_i) = elements i-p .. i (mod n), unwrapped
        e_start = np.arange(N) - space.degree
        U = np.empty((N, tu, da + 1))
        for a in range(tu):
            e = np.mod(e_start + a, n)
            loc = np.mod(np.arange(N) - e, n)  # local index of function i on element e
            U[:, a, :] = u[e, :, loc]
        if not (np.all(np.diff(s_start) == 1) and np.all(counts == tu)):
            raise ConstructionError("circulant path needs unit-step supports")
        if not np.all(ucols == np.mod(np.arange(n)[:, None] + np.arange(space.degree + 1)[None, :], n)):
            raise ConstructionError("unexpected cyclic column layout")
        hinv, K = PC.circulant_inverse(H, n)
        if 2 * K + 1 >= n:
            # the inverse has not decayed within half a period: use one full period
            K = n // 2
            taps = hinv[np.mod(np.arange(-K, K + 1), n)].copy()
            if n % 2 == 0:  # k = -n/2 and +n/2 are the same residue
                taps[0] *= 0.5
                taps[-1] *= 0.5
        else:
            taps = np.concatenate([hinv[-K:] if K else np.empty(0), hinv[: K + 1]])
        nA = da + 1
        nApad = -(-nA // 4) * 4
        ws = s_w.shape[1]
        wspad = -(-ws // 4) * 4
        ktot = tu * nApad + wspad
        uext = np.zeros((N, ktot))
        for a in range(tu):
            uext[:, a * nApad: a * nApad + nA] = 2.0 * U[:, a, :]
        uext[:, tu * nApad: tu * nApad + ws] = -s_w
        zs = nApad + 1
        zs += (4 - zs % 16) % 16
        lp.uext, lp.nApad, lp.zstride = np.ascontiguousarray(uext), nApad, zs
        lp.path = "circulant"
        lp.e_start = e_start.astype(np.int64)
        lp.U = np.ascontiguousarray(U)
        lp.v0 = np.ascontiguousarray(v[0])
        lp.hinv_taps = np.ascontiguousarray(taps)
    else:
        lp.Lb, lp.bw, lp.L21, lp.L22 = PC.fit_cholesky(H, d, fine.closed)
        u_el, u_loc, _ = _incidence(ucols, N)
        v_el, v_loc, _ = _incidence(vcols, fine.dim)
        lp.u, lp.v = np.ascontiguousarray(u), np.ascontiguousarray(v)
        lp.u_el, lp.u_loc, lp.v_el, lp.v_loc = u_el, u_loc, v_el, v_loc
        if graded:
            lp.graded = True
            lp.elh, lp.elm, lp.near_lo, lp.near_cnt = PC.element_pair_geometry(fine)
            lp.ucols, lp.vcols = np.asarray(ucols), np.asarray(vcols)
    disc._logpart = lp
    return lp


# -- device plumbing ------------------------------------------------------------------------


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise DeviceError("PyTorch is required for device memory") from exc
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 assembly has no CPU fallback")
    return torch


def _dev(disc: Discretization, key, make):
    """Per-device cache of the discretization's device data (the current CUDA
    device is part of the key: the multi-GPU host path keeps one copy per GPU)."""
    import torch
    d = disc._dev
    key = (torch.cuda.current_device(), key)
    if key not in d:
        d[key] = make()
    return d[key]


def _to_dev(torch, arr, dtype=None):
    a = np.ascontiguousarray(arr)
    if not a.flags.writeable:
        a = a.copy()
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to("cuda")


def _smooth(disc: Discretization):
    torch = _torch()

    def make():
        rb = disc.rules
        nodes = disc.nodes.nodes
        d = {
            "s": _to_dev(torch, nodes),
            "fx": _to_dev(torch, disc.f_nodes[:, 0]),
            "fy": _to_dev(torch, disc.f_nodes[:, 1]),
            "J": _to_dev(torch, disc.J_nodes),
            "g_start": _to_dev(torch, rb.start.astype(np.int64)),
            "g_w": _to_dev(torch, (rb.weights * disc.J_nodes[np.mod(
                rb.start[:, None] + np.arange(rb.WG)[None, :], len(nodes))])
                * (np.arange(rb.WG)[None, :] < rb.width[:, None])),
            "invp2": _to_dev(torch, disc.invp2) if disc.invp2 is not None else None,
            "near_j2": _to_dev(torch, disc.near_j2) if disc.near_k else None,
            "flag": torch.zeros(1, dtype=torch.int32, device="cuda"),
        }
        st = _lib.WqSmooth(disc.space.dim, len(nodes), rb.WG, int(disc.closed), disc.k1_mode,
                           disc.curve.length, d["s"].data_ptr(), d["fx"].data_ptr(),
                           d["fy"].data_ptr(), d["J"].data_ptr(),
                           d["invp2"].data_ptr() if d["invp2"] is not None else None,
                           d["g_start"].data_ptr(), d["g_w"].data_ptr(), disc.near_k,
                           d["near_j2"].data_ptr() if disc.near_k else None)
        # max node span over output tiles of WQ_TILE rows
        T = _lib.WQ_TILE
        N = disc.space.dim
        first = rb.start[0::T]
        last_idx = np.minimum(np.arange(0, N, T) + T, N) - 1
        span = int((rb.start[last_idx] + rb.WG - first).max())
        d["struct"] = st
        d["span"] = span
        T = _lib.WQ_FTILE
        last_idx = np.minimum(np.arange(0, N, T) + T, N) - 1
        d["span64"] = int((rb.start[last_idx] + rb.WG - rb.start[0::T]).max())
        return d

    return _dev(disc, "smooth", make)


def _check_flag(sm):
    if int(sm["flag"].item()) & _lib.WQ_FLAG_R_NONPOSITIVE:
        sm["flag"].zero_()
        raise GeometryError("R <= 0 on assembly grid")


# band IK1 kernel (sliding windows over per-rule starts) when the tile spans allow it
_IK1_BAND = True


def _k1_vanishes(disc) -> bool:
    """A straight segment traversed at unit parametric speed (degree-1 curve with
    two control points |P1 - P0| = b - a, e.g. the slit of configs 1 and 5):
    |f(s) - f(t)| = |s - t|, so K1 = 1/2 ln(|f(s) - f(t)|^2 / |s - t|^2) vanishes
    identically and IK1 = 0 (geometry.py:225-248 evaluates it to rounding noise,
    max|IK1| ~ 1e-18 of max|A| at config 1)."""
    cb = disc.curve.basis
    P = np.asarray(disc.curve.control_points, dtype=float)
    if cb.degree != 1 or len(P) != 2 or disc.closed:
        return False
    return float(np.hypot(*(P[1] - P[0]))) == float(cb.b - cb.a)


_K1_SHORTCUT = True   # IK1 = 0 on unit-speed straight segments (_k1_vanishes)


def _ik1_skipped(disc) -> bool:
    """IK1 is identically zero and not evaluated (callers then write the log
    part without accumulating, so X is neither zero-filled nor re-read)."""
    return _K1_SHORTCUT and _k1_vanishes(disc)


def _ik1_into(disc, X, accumulate=False, row0=0, row1=None):
    """IK1 (all rows, or rows [row0, row1) x all columns with row0 on a
    64-row tile boundary) into X."""
    torch = _torch()
    sm = _smooth(disc)
    N = disc.space.dim
    row1 = N if row1 is None else row1
    if _K1_SHORTCUT and _k1_vanishes(disc):
        if not accumulate:
            X[: row1 - row0].zero_()     # X points at row0, as for the kernels
        return X
    T = _lib.WQ_FTILE
    if (_IK1_BAND and not accumulate and sm["span64"] <= 144 and 2 <= disc.rules.WG <= 16
            and row0 % T == 0 and (row1 == N or row1 % T == 0)):
        full = row0 == 0 and row1 == N
        _lib.call("wq_ik1_band", ctypes_ref(sm["struct"]), -1 if full else row0 // T,
                  -1 if full else -(-row1 // T), _lib.ptr(X), X.stride(0), sm["span64"],
                  _lib.ptr(sm["flag"]), _lib.stream_handle())
        return X
    _lib.call("wq_ik1", ctypes_ref(sm["struct"]), row0, row1, 0, N, _lib.ptr(X), X.stride(0),
              int(accumulate), sm["span"], _lib.ptr(sm["flag"]), _lib.stream_handle())
    return X


def ctypes_ref(s):
    import ctypes
    return ctypes.byref(s)


# far gaps of the gap table by tiered Gauss orders (30 | 16 | 12) instead of the
# reference's 30 everywhere (quadrature.py:369): same values to rounding
_TIERED_TABLE = True


def _table_rules():
    if _TIERED_TABLE:
        tiers = [PC.gauss_unit(n) for n in PC.GEN_GAUSS_TIERS]
        return (np.concatenate([t[0] for t in tiers]), np.concatenate([t[1] for t in tiers]))
    return PC.gauss_unit(PC.PAIR_FAR_ORDER)


def _table_consts(disc, lp: LogPart):
    """Device copies of the pair table's constant inputs (near-gap unit entries,
    Gauss tiers, centred monomial integrals), uploaded once per discretization."""
    torch = _torch()
    gx, gw = _table_rules()
    return _dev(disc, ("table_consts", _TIERED_TABLE), lambda: [
        _to_dev(torch, lp.near_unit), _to_dev(torch, gx), _to_dev(torch, gw),
        _to_dev(torch, PC.centred_monomial_integrals(lp.da)),
        _to_dev(torch, PC.centred_monomial_integrals(lp.db))])


def _m2_table(disc, lp: LogPart):
    torch = _torch()

    def make():
        n = lp.n_el
        closed = disc.closed
        n_gap = n if closed else 2 * n - 1
        gx, gw = _table_rules()
        m2 = torch.empty((n_gap, lp.da + 1, lp.db + 1), dtype=torch.float64, device="cuda")
        keep = _table_consts(disc, lp)
        _lib.call("wq_pair_table", n, int(closed), lp.da, lp.db, lp.h, _lib.ptr(keep[0]),
                  _lib.ptr(keep[1]), _lib.ptr(keep[2]), len(gx), _lib.ptr(keep[3]),
                  _lib.ptr(keep[4]), _lib.ptr(m2), _lib.stream_handle())
        return m2, keep

    return make()


def _uext_fragments(uext):
    """Uext in the DMMA B-fragment order the x2 kernel reads (include/wqb200.h):
    [row group of 8][k-step of 4 columns][row in group][column in step], rows padded
    with zeros to a multiple of 8, so a warp's fragment is one contiguous 256-byte load."""
    N, ktot = uext.shape
    G = -(-N // 8)
    pad = np.zeros((8 * G, ktot))
    pad[:N] = uext
    return np.ascontiguousarray(pad.reshape(G, 8, ktot // 4, 4).transpose(0, 2, 1, 3))


def _logpart_dev(disc):
    torch = _torch()
    lp = _log_part(disc)

    def make():
        d = {"s_start": _to_dev(torch, lp.s_start.astype(np.int64)),
             "s_w": _to_dev(torch, lp.s_w)}
        N = disc.space.dim
        if lp.path == "circulant":
            d["e_start"] = _to_dev(torch, lp.e_start)
            d["U"] = _to_dev(torch, lp.U)
            d["v0"] = _to_dev(torch, lp.v0)
            d["taps"] = _to_dev(torch, lp.hinv_taps)
            d["uext"] = _to_dev(torch, _uext_fragments(lp.uext))
            tu = lp.U.shape[1]
            d["struct"] = _lib.WqLogpart(N, lp.n_el, lp.da, tu, lp.s_w.shape[1],
                                         d["e_start"].data_ptr(), d["U"].data_ptr(),
                                         d["s_start"].data_ptr(), d["s_w"].data_ptr())
        else:
            NE = disc.refined.basis.dim
            for k in ("u", "v", "u_el", "u_loc", "v_el", "v_loc", "Lb", "L21", "L22",
                      "elh", "elm", "near_lo", "near_cnt"):
                if getattr(lp, k) is not None:
                    d[k] = _to_dev(torch, getattr(lp, k))
            if lp.graded:
                tiers = [PC.gauss_unit(n) for n in PC.GEN_GAUSS_TIERS]
                d["gx"] = _to_dev(torch, np.concatenate([t[0] for t in tiers]))
                d["gw"] = _to_dev(torch, np.concatenate([t[1] for t in tiers]))
                d["touch"] = _to_dev(torch, PC.touch_rules())
                d["near_unit"] = _to_dev(torch, lp.near_unit)
                d["ca"] = _to_dev(torch, PC.centred_monomial_integrals(lp.da))
                d["cb"] = _to_dev(torch, PC.centred_monomial_integrals(lp.db))
            d["struct"] = _lib.WqLogpart(N, NE, lp.da, 0, lp.s_w.shape[1], None, None,
                                         d["s_start"].data_ptr(), d["s_w"].data_ptr())
        return d

    return lp, _dev(disc, "logpart", make)


def _circ_tables(disc):
    """Pair table -> folded circulant tables (Z' = H^{-1}-folded Theta gap
    table, ff = H^{-1} D H^{-1}) on the device; O(n_el) work per call."""
    torch = _torch()
    lp, d = _logpart_dev(disc)
    st = _lib.stream_handle()
    m2, keep = _m2_table(disc, lp)
    n = lp.n_el
    nA = lp.da + 1
    Zp = torch.empty((n, nA), dtype=torch.float64, device="cuda")
    Zw = torch.empty((n, nA), dtype=torch.float64, device="cuda")
    ff = torch.empty(n, dtype=torch.float64, device="cuda")
    work = torch.empty(n, dtype=torch.float64, device="cuda")
    K = (len(lp.hinv_taps) - 1) // 2
    _lib.call("wq_circ_tables", n, lp.da, lp.db, _lib.ptr(m2), _lib.ptr(d["v0"]),
              _lib.ptr(d["taps"]), K, _lib.ptr(Zp), _lib.ptr(ff), _lib.ptr(work), _lib.ptr(Zw), st)
    return Zp, ff


def _ik2_x2_rows(disc, X, row0, row1, accumulate=True, tables=None):
    """Circulant path: X[rows] (+)= X2[row0:row1, :] (X points at row0)."""
    lp, d = _logpart_dev(disc)
    N = disc.space.dim
    Zp, ff = _circ_tables(disc) if tables is None else tables
    _lib.call("wq_ik2_circ", ctypes_ref(d["struct"]), _lib.ptr(Zp), _lib.ptr(ff), row0, row1, 0, N,
              _lib.ptr(X), X.stride(0), int(accumulate), _lib.stream_handle())
    return X


def _ik2_x2_into(disc, X, accumulate=True, sym_alpha=None):
    """X (+)= X2 (circulant: X2 itself; general: X2^T -- callers symmetrise).
    With sym_alpha the symmetrisation is included: X <- sym_alpha (X' + X'^T),
    X' = (X if accumulate) + X2 (general path: fused into the last kernel)."""
    torch = _torch()
    lp, d = _logpart_dev(disc)
    N = disc.space.dim
    st = _lib.stream_handle()
    if lp.path == "circulant":
        _ik2_x2_rows(disc, X, 0, N, accumulate)
        if sym_alpha is not None:
            _lib.call("wq_symmetrize", _lib.ptr(X), N, sym_alpha, st)
        return X
    NE = disc.refined.basis.dim
    thetaT, D = _theta_d(disc, lp, d)
    # Phi = H^{-1} (2 Theta^T - D H^{-1} S)  (= 2 H^{-1} Theta^T - F S, F = H^{-1} D H^{-1}:
    # one banded solve fewer than forming F); D H^{-1} = (H^{-1} D)^T is read transposed
    # from H^{-1} D when the band rows of a 64-column block fit in shared memory
    span = _s_band_span(lp)
    if span * 33 * 8 <= 200 * 1024 and lp.s_w.shape[1] <= 20:
        _hsolver(lp, d, NE)(D, NE)
        _lib.call("wq_gather_yts", ctypes_ref(d["struct"]), 2.0, _lib.ptr(D), _lib.ptr(thetaT),
                  span, st)
    else:
        E = _fit_dh(disc, lp, d, D)
        _lib.call("wq_gather_fs", ctypes_ref(d["struct"]), 2.0, _lib.ptr(E), _lib.ptr(thetaT), st)
    _hsolver(lp, d, NE)(thetaT, N)
    # X[j][i] (+)= sum_m S[m, j] Phi[m, i]  (= X2^T)
    if sym_alpha is not None and X.stride(0) == N:
        _lib.call("wq_st_phi_sym", ctypes_ref(d["struct"]), _lib.ptr(thetaT), _lib.ptr(X),
                  sym_alpha, int(accumulate), st)
        return X
    _lib.call("wq_add_st_phi", ctypes_ref(d["struct"]), _lib.ptr(thetaT), 0, N, _lib.ptr(X),
              X.stride(0), int(accumulate), st)
    if sym_alpha is not None:
        _lib.call("wq_symmetrize", _lib.ptr(X), N, sym_alpha, st)
    return X


def _theta_d(disc, lp: LogPart, d, rows=None, want_theta=True, want_d=True):
    """Theta^T (all columns, or the block rows = (row0, row1)) and D; either
    may be skipped (None): a rank's row block needs only its Theta^T columns,
    D is computed once per assembly (general_prepare)."""
    torch = _torch()
    st = _lib.stream_handle()
    N, NE = disc.space.dim, disc.refined.basis.dim
    if lp.graded:
        return _graded_theta_d(disc, lp, d, rows, want_theta, want_d)
    m2, keep = _m2_table(disc, lp)
    pp = _lib.WqPairs(N, NE, lp.n_el, m2.shape[0], lp.da, lp.db, int(disc.closed),
                      lp.u_el.shape[1], lp.v_el.shape[1], d["u_el"].data_ptr(),
                      d["u_loc"].data_ptr(), d["v_el"].data_ptr(), d["v_loc"].data_ptr(),
                      d["u"].data_ptr(), disc.space.degree, d["v"].data_ptr(),
                      m2.data_ptr())
    thetaT = D = None
    if want_theta:
        r0, r1 = (0, N) if rows is None else rows
        thetaT = torch.empty((NE, r1 - r0), dtype=torch.float64, device="cuda")
        _lib.call("wq_theta_t_rows", ctypes_ref(pp), r0, r1, _lib.ptr(thetaT), r1 - r0, st)
    if want_d:
        D = torch.empty((NE, NE), dtype=torch.float64, device="cuda")
        _lib.call("wq_dmat", ctypes_ref(pp), _lib.ptr(D), st)
    return thetaT, D


# segmented banded solves (columns x row segments in parallel) from this many rows on
_SEG_ROWS = 1024
_SEG_MIN_N = 2048


def _seg_warmup(lp: LogPart) -> int:
    """Warm-up rows of the segmented solves: the measured decay length of the
    factor's inverse to 1e-20 (precompute.inverse_decay_rows) plus a margin,
    or -1 (sequential solves) when it does not decay within 2048 rows."""
    if lp.seg_k0 is None:
        k = PC.inverse_decay_rows(lp.Lb, lp.bw)
        lp.seg_k0 = -1 if k < 0 else -(-(k + 32) // 16) * 16
    return lp.seg_k0


def _hsolver(lp: LogPart, d, NE):
    """Y <- H^{-1} Y on ncols columns (banded / arrow Cholesky of the fit)."""
    st = _lib.stream_handle()

    def hsolve(Y, ncols):
        k0 = _seg_warmup(lp) if lp.L21 is None and lp.bw <= 8 and NE >= _SEG_MIN_N else -1
        if k0 >= 0:
            torch = _torch()
            nseg = -(-NE // _SEG_ROWS)
            state = torch.empty(max(1, (nseg - 1) * lp.bw * ncols), dtype=torch.float64,
                                device="cuda")
            _lib.call("wq_band_solve_seg", NE, lp.bw, _lib.ptr(d["Lb"]), _lib.ptr(Y), ncols,
                      Y.stride(0), _SEG_ROWS, k0, _lib.ptr(state), st)
        elif lp.L21 is None and lp.bw <= 8:
            _lib.call("wq_band_solve_win", NE, lp.bw, _lib.ptr(d["Lb"]), _lib.ptr(Y), ncols,
                      Y.stride(0), st)
        elif lp.L21 is None:
            _lib.call("wq_band_solve_cols", NE, lp.bw, _lib.ptr(d["Lb"]), _lib.ptr(Y), ncols,
                      Y.stride(0), st)
        else:
            _lib.call("wq_cyc_solve_cols", NE, lp.bw, _lib.ptr(d["Lb"]), _lib.ptr(d["L21"]),
                      _lib.ptr(d["L22"]), _lib.ptr(Y), ncols, Y.stride(0), st)
    return hsolve


def _s_band_span(lp: LogPart) -> int:
    """Fit rows touched by the S bands of 64 consecutive columns (wq_gather_yts)."""
    if lp.s_span is None:
        ss = np.asarray(lp.s_start, dtype=np.int64)
        i0 = np.arange(0, len(ss), 64)
        i1 = np.minimum(i0 + 63, len(ss) - 1)
        lp.s_span = int((ss[i1] - ss[i0]).max()) + int(lp.s_w.shape[1])
    return lp.s_span


def _fit_dh(disc, lp: LogPart, d, D):
    """E = D H^{-1} = (H^{-1} D)^T, D symmetric (D is overwritten by H^{-1} D).  The fit term
    C^T D C = S^T (H^{-1} D H^{-1}) S enters Phi as H^{-1} (E S), so the second solve of
    F = H^{-1} D H^{-1} merges with the solve of Theta^T (assembly.py:233-245 in X-form)."""
    torch = _torch()
    NE = disc.refined.basis.dim
    _hsolver(lp, d, NE)(D, NE)
    E = torch.empty_like(D)
    _lib.call("wq_transpose", _lib.ptr(D), NE, NE, _lib.ptr(E), _lib.stream_handle())
    return E


def general_prepare(disc):
    """E = D H^{-1} of the general path (replicated per rank; computed once per
    assembly and shared by its row blocks)."""
    lp, d = _logpart_dev(disc)
    _, D = _theta_d(disc, lp, d, want_theta=False)
    return _fit_dh(disc, lp, d, D)


def general_rows_into(disc, X_rows, row0: int, row1: int, F=None):
    """Rows [row0, row1) of the unsymmetrised X = IK1 + X2 of the general
    (non-circulant) path into X_rows (leading dimension N): IK1 rows, the
    block's Theta^T columns, replicated D and E = D H^{-1} (passed as F),
    Phi = H^{-1} (2 Theta^T - E S) on the block's columns,
    X2[i][j] = sum_t S_j[t] Phi[s_j + t][i].  No communication."""
    lp, d = _logpart_dev(disc)
    sm = _smooth(disc)
    st = _lib.stream_handle()
    N, NE = disc.space.dim, disc.refined.basis.dim
    nr = row1 - row0
    skip = _ik1_skipped(disc)
    if not skip:
        _ik1_into(disc, X_rows, accumulate=False, row0=row0, row1=row1)
    if F is None:
        F = general_prepare(disc)
    T, _ = _theta_d(disc, lp, d, rows=(row0, row1), want_d=False)
    _lib.call("wq_gather_fs_rows", ctypes_ref(d["struct"]), 2.0, _lib.ptr(F), _lib.ptr(T), row0,
              row1, nr, st)
    _hsolver(lp, d, NE)(T, nr)
    torch = _torch()
    PhiT = torch.empty((nr, NE), dtype=torch.float64, device="cuda")
    _lib.call("wq_transpose", _lib.ptr(T), NE, nr, _lib.ptr(PhiT), st)
    _lib.call("wq_phi_s_rows", ctypes_ref(d["struct"]), _lib.ptr(PhiT), row0, row1,
              _lib.ptr(X_rows), X_rows.stride(0), 0 if skip else 1, st)
    return X_rows


# device bytes for one chunk of per-pair Theta / D blocks (graded meshes)
_GEN_CHUNK_BYTES = 1 << 30
# graded open meshes: read far pairs of equal widths from the unit gap table
_GEN_GAP_TABLE = True


def _gap_table(disc, lp: LogPart, h0: float):
    """The reference's gap-indexed pair table (quadrature.py:441-504) for an
    open mesh of n_el elements of width h0 (device, wq_pair_table; h0 = 1
    gives the unit moments M')."""
    torch = _torch()
    n = lp.n_el
    gx, gw = _table_rules()
    m2 = torch.empty((2 * n - 1, lp.da + 1, lp.db + 1), dtype=torch.float64, device="cuda")
    keep = _table_consts(disc, lp)
    _lib.call("wq_pair_table", n, 0, lp.da, lp.db, h0, _lib.ptr(keep[0]), _lib.ptr(keep[1]),
              _lib.ptr(keep[2]), len(gx), _lib.ptr(keep[3]), _lib.ptr(keep[4]), _lib.ptr(m2),
              _lib.stream_handle())
    return m2


# graded open meshes: lattice route (Theta / D straight from the gap table for
# outer elements on the width-h0 lattice) when at most this many elements are off it
_LATTICE_MAX_OFF = 4096
_LATTICE_MAX_BYTES = 8 << 30   # device bytes of the lattice route's off-lattice moments
# D by its lower storage triangle + mirror (D is symmetric)
_YS_SYM_D = True
_NOT_LATTICE = np.iinfo(np.int64).min


def lattice_classes(elh, elm):
    """Elements on the lattice of the median width h0 (width within 2e-11,
    centre on the h0 grid to 1e-10 relative): returns (kidx, gidx, glist), kidx
    the lattice index (or int64 min), gidx the index among the others (or -1).
    The tolerances are tighter than the per-pair snap (1e-10 width, 1e-9
    offset), so every lattice pair is one the reference's table recipe covers."""
    h0 = float(np.median(elh))
    on = np.abs(elh / h0 - 1.0) < 2e-11
    kidx = np.full(len(elh), _NOT_LATTICE, np.int64)
    if on.any():
        ref = elm[np.argmax(on)]
        k = (elm - ref) / h0
        kr = np.rint(k)
        on &= np.abs(k - kr) < 1e-10 * np.maximum(1.0, np.abs(k))
        kidx[on] = kr[on].astype(np.int64)
    glist = np.flatnonzero(~on).astype(np.int64)
    gidx = np.full(len(elh), -1, np.int32)
    gidx[glist] = np.arange(len(glist), dtype=np.int32)
    return kidx, gidx, glist


_YS_MMA = True        # pure-lattice 64 x 64 tiles of the Y-stage on DMMA (wq_ystage_mma)
_YM_T, _YM_FSP, _YM_ESP, _YM_ZR, _YM_TFRONT = 64, 72, 68, 152, 8
_YM_NOT_PURE = -2 ** 31


def _ym_tiles(lo, hi, ko_el, start, stop, rows):
    """Per 64-function tile from ``start``: the common lattice offset k_e - e of every
    element the tile's supports touch, or INT32_MIN when the tile is partial, leaves
    the lattice, changes offset, or exceeds the tensor-core kernel's spans (row tiles:
    first elements within 68; column tiles: at most 72 elements)."""
    out = []
    for t0 in range(start, stop, _YM_T):
        t1 = t0 + _YM_T - 1
        ok = t1 < stop
        if ok:
            ea, eb = int(lo[t0]), int(hi[t1])
            ks = ko_el[ea: eb + 1]
            ok = bool(np.all(ks == ks[0])) and ks[0] != _YM_NOT_PURE
            span_ok = (int(lo[t1]) - ea <= _YM_ESP) if rows else (eb - ea + 1 <= _YM_FSP)
            ok = ok and span_ok
        out.append(int(ko_el[int(lo[t0])]) if ok else _YM_NOT_PURE)
    return np.asarray(out, np.int32)


def _ys_tile_list(row_ko, col_ko, n_rows, n_cols, sym):
    """(16-row tile, 64-column tile) pairs left to wq_ystage once wq_ystage_mma owns the
    tiles with equal pure offsets; ``sym``: only tiles meeting the storage triangle
    (last column >= first row).  int32 (n, 2)."""
    nrt = -(-n_rows // 16)
    nct = -(-n_cols // _YM_T)
    rk = np.repeat(np.asarray(row_ko, np.int64), _YM_T // 16)[:nrt]
    ck = np.asarray(col_ko, np.int64)[:nct]
    todo = ~((rk[:, None] != _YM_NOT_PURE) & (rk[:, None] == ck[None, :]))
    if sym:
        r0 = 16 * np.arange(nrt)[:, None]
        c_last = np.minimum(_YM_T * (np.arange(nct)[None, :] + 1), n_cols) - 1
        todo &= c_last >= r0
    return np.ascontiguousarray(np.argwhere(todo).astype(np.int32))


def _support_ranges(el):
    """First / last element of each function's support from a (-1 padded)
    incidence array (open meshes: contiguous)."""
    big = np.iinfo(np.int64).max
    lo = np.where(el >= 0, el, big).min(axis=1)
    hi = np.where(el >= 0, el, -1).max(axis=1)
    return lo.astype(np.int64), hi.astype(np.int64)


def _tile_span(lo, hi, tile):
    n = len(lo)
    starts = np.arange(0, n, tile)
    ends = np.minimum(starts + tile, n) - 1
    return int((hi[ends] - lo[starts] + 1).max())


def _graded_theta_d(disc, lp: LogPart, d, rows=None, want_theta=True, want_d=True):
    """Theta^T (N_E x N, or N_E x (row1 - row0) for rows = (row0, row1)) and D
    (N_E x N_E) of a graded mesh (either may be skipped)."""
    consecutive = all(np.array_equal(c, c[:, :1] + np.arange(c.shape[1])[None, :])
                      for c in (lp.ucols, lp.vcols))     # element functions are consecutive rows
    if not disc.closed and _GEN_GAP_TABLE and lp.db == 4 and consecutive:
        kidx, gidx, glist = lattice_classes(lp.elh, lp.elm)
        # the off-lattice moments (len(glist), n_el, P+1, d+1) stay within a byte budget
        mg_bytes = len(glist) * lp.n_el * (lp.da + 1) * (lp.db + 1) * 8
        if len(glist) <= _LATTICE_MAX_OFF and mg_bytes <= _LATTICE_MAX_BYTES:
            return _lattice_theta_d(disc, lp, d, kidx, gidx, glist, rows, want_theta, want_d)
    return _blocks_theta_d(disc, lp, d, rows=rows, want_theta=want_theta, want_d=want_d)


def _lattice_theta_d(disc, lp: LogPart, d, kidx, gidx, glist, rows=None, want_theta=True,
                     want_d=True):
    """Theta^T and D of a graded open mesh: lattice outer elements straight
    from the unit gap table (wq_ystage), the few others by the block route
    (either output may be skipped: None)."""
    torch = _torch()
    st = _lib.stream_handle()
    N, NE, n = disc.space.dim, disc.refined.basis.dim, lp.n_el
    nU, nB = lp.u.shape[2], lp.db + 1
    da1 = lp.da + 1
    key = "lattice"
    if key not in d:
        u_lo, u_hi = _support_ranges(lp.u_el)
        v_lo, v_hi = _support_ranges(lp.v_el)
        d[key] = {
            "kidx": _to_dev(torch, kidx), "gidx": _to_dev(torch, gidx),
            "glist": _to_dev(torch, glist) if len(glist) else None,
            "u_lo": _to_dev(torch, u_lo), "u_hi": _to_dev(torch, u_hi),
            "v_lo": _to_dev(torch, v_lo), "v_hi": _to_dev(torch, v_hi),
            "u_es": _tile_span(u_lo, u_hi, 16), "v_es": _tile_span(v_lo, v_hi, 16),
            "v_fs": _tile_span(v_lo, v_hi, 64),
            "ucols": _to_dev(torch, lp.ucols.astype(np.int64)),
            "vcols": _to_dev(torch, lp.vcols.astype(np.int64)),
        }
    L = d[key]
    m2u = _gap_table(disc, lp, 1.0)
    mgc = None
    max_near = int(lp.near_cnt.max())
    if len(glist):
        mgc = torch.zeros((len(glist), n, da1, nB), dtype=torch.float64, device="cuda")
        _lib.call("wq_gen_moments_far", n, da1, nB, len(glist), _lib.ptr(L["glist"]),
                  _lib.ptr(L["gidx"]), _lib.ptr(d["elh"]), _lib.ptr(d["elm"]),
                  _lib.ptr(d["near_lo"]), _lib.ptr(d["near_cnt"]), _lib.ptr(d["gx"]),
                  _lib.ptr(d["gw"]), _lib.ptr(mgc), st)
        _lib.call("wq_gen_near_moments", n, lp.da, lp.db, _lib.ptr(d["elh"]), _lib.ptr(d["elm"]),
                  _lib.ptr(d["near_lo"]), _lib.ptr(d["near_cnt"]), max_near,
                  _lib.ptr(d["near_unit"]), _lib.ptr(d["touch"]), _lib.ptr(d["ca"]),
                  _lib.ptr(d["cb"]), _lib.ptr(L["gidx"]), _lib.ptr(mgc), st)
    r0, r1 = (0, N) if rows is None else rows
    thetaT = torch.empty((NE, r1 - r0), dtype=torch.float64, device="cuda") if want_theta else None
    D = torch.empty((NE, NE), dtype=torch.float64, device="cuda") if want_d else None
    mg = _lib.ptr(mgc) if mgc is not None else None
    wc = lp.v_el.shape[1]
    cols = (_lib.ptr(d["v_el"]), _lib.ptr(d["v_loc"]), _lib.ptr(L["v_lo"]), _lib.ptr(L["v_hi"]))
    tail = (_lib.ptr(d["v"]), nB, _lib.ptr(d["elh"]), _lib.ptr(L["kidx"]), _lib.ptr(L["gidx"]),
            _lib.ptr(m2u), da1, mg, _lib.ptr(d["ca"]), _lib.ptr(d["cb"]))
    mma = _YS_MMA and r0 % _YM_T == 0 and nU == 5 and nB == 5 and da1 == 17 and wc <= 5
    kT = kD = kC = None
    listT = listD = (None, 0)
    if mma:
        mkey = ("ym", r0, r1)
        if mkey not in L:
            ko_el = np.where(kidx != _NOT_LATTICE, kidx - np.arange(n), _YM_NOT_PURE)
            u_lo, u_hi = _support_ranges(lp.u_el)
            v_lo, v_hi = _support_ranges(lp.v_el)
            tT = _ym_tiles(u_lo, u_hi, ko_el, r0, r1, True)
            tD = _ym_tiles(v_lo, v_hi, ko_el, 0, NE, True)
            tC = _ym_tiles(v_lo, v_hi, ko_el, 0, NE, False)
            L[mkey] = {"T": _to_dev(torch, tT), "D": _to_dev(torch, tD), "C": _to_dev(torch, tC),
                       # the tiles left to the CUDA-core kernel (a few per cent)
                       "listT": _to_dev(torch, _ys_tile_list(tT, tC, r1 - r0, NE, False)),
                       "listD": _to_dev(torch, _ys_tile_list(tD, tC, NE, NE, bool(_YS_SYM_D)))}
        Y = L[mkey]
        kT, kD, kC = _lib.ptr(Y["T"]), _lib.ptr(Y["D"]), _lib.ptr(Y["C"])
        listT = (_lib.ptr(Y["listT"]), Y["listT"].shape[0])
        listD = (_lib.ptr(Y["listD"]), Y["listD"].shape[0])
        n_tab = 2 * n - 1 + _YM_ZR + _YM_TFRONT
        f64 = dict(dtype=torch.float64, device="cuda")
        kpT, kpD = -(-5 * da1 // 4) * 4, -(-5 * nB // 4) * 4
        Tb = torch.empty((5, n_tab, 20), **f64)
        vsum = torch.empty((NE, 5), **f64)
        common = (_lib.ptr(d["v_el"]), _lib.ptr(d["v_loc"]))
        mcols = common + (_lib.ptr(L["v_lo"]), _lib.ptr(L["v_hi"]), _lib.ptr(d["v"]))
        # per-column-tile incidence tables of the contraction warps (TMA, a tile ahead)
        CvT = torch.empty((NE // _YM_T, _YM_T * 25), **f64)
        CiT = torch.empty((NE // _YM_T, _YM_T * 5), dtype=torch.int32, device="cuda")
        _lib.call("wq_ystage_mma_tiles", NE, wc, *common, _lib.ptr(L["v_lo"]), _lib.ptr(d["v"]),
                  _lib.ptr(CvT), _lib.ptr(CiT), st)
        ctabs = (_lib.ptr(CvT), _lib.ptr(CiT))
        if want_theta:      # (the first prep also re-lays the table out: Tb)
            CrT, LtT = torch.empty((5, -(-N // 8) * 8, kpT), **f64), torch.empty((N, 5), **f64)
            _lib.call("wq_ystage_mma_prep", N, NE, n, da1, nU, wc, _lib.ptr(L["ucols"]),
                      _lib.ptr(L["u_lo"]), _lib.ptr(L["u_hi"]), *common, _lib.ptr(d["u"]), da1,
                      _lib.ptr(d["v"]), _lib.ptr(d["elh"]), _lib.ptr(m2u), da1, _lib.ptr(d["ca"]),
                      _lib.ptr(d["cb"]), _lib.ptr(CrT), _lib.ptr(LtT), _lib.ptr(vsum),
                      _lib.ptr(Tb), n_tab, st)
        if want_d:
            CrD, LtD = torch.empty((5, -(-NE // 8) * 8, kpD), **f64), torch.empty((NE, 5), **f64)
            tb = None if want_theta else _lib.ptr(Tb)
            _lib.call("wq_ystage_mma_prep", NE, NE, n, nB, nB, wc, _lib.ptr(L["vcols"]),
                      _lib.ptr(L["v_lo"]), _lib.ptr(L["v_hi"]), *common, _lib.ptr(d["v"]), nB,
                      _lib.ptr(d["v"]), _lib.ptr(d["elh"]), None if tb is None else _lib.ptr(m2u),
                      da1, _lib.ptr(d["ca"]), _lib.ptr(d["cb"]), _lib.ptr(CrD), _lib.ptr(LtD),
                      _lib.ptr(vsum), tb, n_tab, st)
        if want_theta:
            _lib.call("wq_ystage_mma", N, NE, n, da1, wc, _lib.ptr(L["u_lo"]), *mcols,
                      _lib.ptr(CrT), _lib.ptr(LtT), _lib.ptr(vsum), *ctabs, _lib.ptr(Tb), n_tab,
                      kT, kC, _lib.ptr(thetaT), r1 - r0, r0, r1, 0, st)
        if want_d:
            _lib.call("wq_ystage_mma", NE, NE, n, nB, wc, _lib.ptr(L["v_lo"]), *mcols,
                      _lib.ptr(CrD), _lib.ptr(LtD), _lib.ptr(vsum), *ctabs, _lib.ptr(Tb), n_tab,
                      kD, kC, _lib.ptr(D), NE, 0, NE, int(_YS_SYM_D), st)
    # (with the tensor-core tiles taken out, an empty list means nothing is left)
    if want_theta and not (mma and listT[1] == 0):
        _lib.call("wq_ystage", N, NE, n, da1, nU, wc, _lib.ptr(L["ucols"]),
                  _lib.ptr(L["u_lo"]), _lib.ptr(L["u_hi"]), *cols, _lib.ptr(d["u"]), da1, *tail,
                  L["v_fs"], L["u_es"], _lib.ptr(thetaT), r1 - r0, r0, r1, 0, kT, kC, *listT, st)
    if want_d and not (mma and listD[1] == 0):
        _lib.call("wq_ystage", NE, NE, n, nB, nB, wc, _lib.ptr(L["vcols"]),
                  _lib.ptr(L["v_lo"]), _lib.ptr(L["v_hi"]), *cols, _lib.ptr(d["v"]), nB, *tail,
                  L["v_fs"], L["v_es"], _lib.ptr(D), NE, 0, NE, int(_YS_SYM_D), kD, kC, *listD, st)
    if len(glist):
        _blocks_theta_d(disc, lp, d, outer=glist, thetaT=thetaT, D=D, rows=rows,
                        want_theta=want_theta, want_d=want_d)
    # D's lower storage triangle is complete (lattice + block parts): mirror it
    if want_d and _YS_SYM_D:
        # (the tensor-core tiles wrote their mirrors themselves: row_ko / col_ko skip them)
        _lib.call("wq_mirror_lower", _lib.ptr(D), NE, NE, kD, kC, st)
    return thetaT, D


def _blocks_theta_d(disc, lp: LogPart, d, outer=None, thetaT=None, D=None, rows=None,
                    want_theta=True, want_d=True):
    """Theta^T (N_E x N) and D (N_E x N_E) of a graded mesh: per-pair blocks
    for chunks of outer elements (all of them, or the runs of ``outer``), then
    deterministic gathers, accumulating into ``thetaT`` / ``D`` when given
    (replaces the gap-table accumulation of assembly.py:206-236, which the
    reference only supports on uniform meshes)."""
    torch = _torch()
    st = _lib.stream_handle()
    N, NE, n = disc.space.dim, disc.refined.basis.dim, lp.n_el
    nU, nB = lp.u.shape[2], lp.db + 1
    per_e = n * (nU * nB + nB * nB) * 8
    chunk = int(min(n, max(64, _GEN_CHUNK_BYTES // per_e // 64 * 64)))   # whole 64-element tiles
    wt = torch.empty((n, nU, nB, chunk), dtype=torch.float64, device="cuda")   # chunk-minor
    wd = torch.empty((n, nB, nB, chunk), dtype=torch.float64, device="cuda")
    flags = torch.empty((n, -(-chunk // 64)), dtype=torch.int32, device="cuda")
    r0, r1 = (0, N) if rows is None else rows
    if outer is None:
        thetaT = torch.zeros((NE, r1 - r0), dtype=torch.float64, device="cuda") if want_theta else None
        D = torch.zeros((NE, NE), dtype=torch.float64, device="cuda") if want_d else None
        ranges = [(e0, min(n, e0 + chunk)) for e0 in range(0, n, chunk)]
    else:   # contiguous runs of the listed outer elements, split into chunks
        cuts = np.flatnonzero(np.diff(outer) != 1) + 1
        ranges = []
        for run in np.split(outer, cuts):
            for a in range(int(run[0]), int(run[-1]) + 1, chunk):
                ranges.append((a, min(int(run[-1]) + 1, a + chunk)))
    max_near = int(lp.near_cnt.max())
    period = float(disc.refined.basis.length) if disc.closed else 0.0
    # open meshes: the reference's unit gap table serves every far pair of
    # equal widths at an integer offset (scaled per pair by the width)
    m2u = _gap_table(disc, lp, 1.0) if (not disc.closed and _GEN_GAP_TABLE
                                        and outer is None) else None
    wu, wv = lp.u_el.shape[1], lp.v_el.shape[1]
    for e0, e1 in ranges:
        _lib.call("wq_gen_pair_blocks", n, e0, e1, lp.da, lp.db, nU - 1, int(disc.closed), period,
                  _lib.ptr(d["elh"]), _lib.ptr(d["elm"]), _lib.ptr(d["u"]), _lib.ptr(d["v"]),
                  _lib.ptr(d["near_lo"]), _lib.ptr(d["near_cnt"]), max_near,
                  _lib.ptr(d["near_unit"]), _lib.ptr(d["touch"]), _lib.ptr(d["gx"]),
                  _lib.ptr(d["gw"]), _lib.ptr(m2u) if m2u is not None else None,
                  _lib.ptr(d["ca"]), _lib.ptr(d["cb"]), _lib.ptr(wt),
                  _lib.ptr(wd), chunk, _lib.ptr(flags), st)
        uc, vc = lp.ucols[e0:e1], lp.vcols[e0:e1]
        i0, i1 = max(int(uc.min()), r0), min(int(uc.max()) + 1, r1)
        if want_theta and i1 > i0:
            _lib.call("wq_gen_gather_theta", N, NE, e0, e1, chunk, i0, i1, wu, wv, nU, nB,
                      _lib.ptr(d["u_el"]), _lib.ptr(d["u_loc"]), _lib.ptr(d["v_el"]),
                      _lib.ptr(d["v_loc"]), _lib.ptr(wt), _lib.ptr(thetaT), r1 - r0, r0, st)
        if want_d:
            _lib.call("wq_gen_gather_d", NE, e0, e1, chunk, int(vc.min()), int(vc.max()) + 1, wv,
                      nB, _lib.ptr(d["v_el"]), _lib.ptr(d["v_loc"]), _lib.ptr(wd), _lib.ptr(D), st)
    return thetaT, D


def _new_square(disc):
    torch = _torch()
    N = disc.space.dim
    return torch.empty((N, N), dtype=torch.float64, device="cuda")


def _zext_table(disc):
    """Z' and ff packed into the row layout the DMMA kernel streams."""
    torch = _torch()
    lp, d = _logpart_dev(disc)
    Zp, ff = _circ_tables(disc)
    n = lp.n_el
    Zext = torch.empty((n, lp.zstride), dtype=torch.float64, device="cuda")
    _lib.call("wq_zext", n, lp.da + 1, lp.nApad, lp.zstride, _lib.ptr(Zp), _lib.ptr(ff),
              _lib.ptr(Zext), _lib.stream_handle())
    return Zext


_AUX_STREAMS = {}


def _aux_stream(torch):
    dev = torch.cuda.current_device()
    if dev not in _AUX_STREAMS:
        _AUX_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return _AUX_STREAMS[dev]


def pair_chunks(N: int, chunks: int):
    """Split the upper-triangle tile pairs (64-row tiles) into contiguous
    ranges of about equal size."""
    nb = -(-N // _lib.WQ_FTILE)
    total = nb * (nb + 1) // 2
    chunks = max(1, min(chunks, total))
    edges = np.linspace(0, total, chunks + 1).round().astype(np.int64)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def _assemble_v2(disc: Discretization, X, alpha: float, w_ik1: float = 2.0, zext=None,
                 chunks: int = None):
    """Circulant pipeline in place in X: tables -> ik1_sym (upper tiles of IK1)
    -> x2_pairs (DMMA log part + fused symmetric epilogue).  The tile pairs are
    split into chunks; IK1 chunks run on an auxiliary stream and the x2 chunk k
    waits only for IK1 chunk k, so the FP64 (ik1) and FP64-tensor (x2) kernels
    of neighbouring chunks overlap on the SMs."""
    torch = _torch()
    lp, d = _logpart_dev(disc)
    sm = _smooth(disc)
    main = torch.cuda.current_stream()
    st = _lib.stream_handle(main)
    N = disc.space.dim
    if chunks is None:
        chunks = 1
    ranges = pair_chunks(N, chunks)
    ik1_first = zext is None and w_ik1 != 0.0 and len(ranges) == 1
    if ik1_first:
        # IK1 does not need the gap tables: they build on an auxiliary stream while
        # the IK1 tiles run, and x2 waits for both
        aux = _aux_stream(torch)
        aux.wait_stream(main)          # before the IK1 launch: the tables overlap it
        _lib.call("wq_ik1_sym", ctypes_ref(sm["struct"]), _lib.ptr(X), X.stride(0), sm["span64"],
                  _lib.ptr(sm["flag"]), st)
        with torch.cuda.stream(aux):
            Zext = _zext_table(disc)
        Zext.record_stream(main)
        main.wait_stream(aux)
    else:
        Zext = _zext_table(disc) if zext is None else zext
    x2args = (N, disc.space.degree, lp.da + 1, lp.nApad, lp.s_w.shape[1], lp.uext.shape[1],
              lp.zstride, _lib.ptr(d["uext"]), _lib.ptr(Zext), _lib.ptr(d["s_w"]), alpha, w_ik1)
    if w_ik1 == 0.0:
        _lib.call("wq_x2_pairs", *x2args, _lib.ptr(X), X.stride(0), st)
        return X
    if len(ranges) == 1:
        if not ik1_first:
            _lib.call("wq_ik1_sym", ctypes_ref(sm["struct"]), _lib.ptr(X), X.stride(0),
                      sm["span64"], _lib.ptr(sm["flag"]), st)
        _lib.call("wq_x2_pairs", *x2args, _lib.ptr(X), X.stride(0), st)
        return X
    aux = _aux_stream(torch)
    aux.wait_stream(main)
    ast = _lib.stream_handle(aux)
    events = []
    for a, b in ranges:
        _lib.call("wq_ik1_pairs", ctypes_ref(sm["struct"]), a, b, _lib.ptr(X), X.stride(0),
                  _lib.ptr(sm["flag"]), ast)
        ev = torch.cuda.Event()
        ev.record(aux)
        events.append(ev)
    for (a, b), ev in zip(ranges, events):
        main.wait_event(ev)
        _lib.call("wq_x2_pairs_range", *x2args, a, b, _lib.ptr(X), X.stride(0), st)
    return X


def _use_v2(disc) -> bool:
    """The v2/v3 tile kernels need the circulant log part and the closed
    uniform rule layout (rule i on nodes 2(i-p)+1 .. 2(i-p)+2p+1)."""
    lp = _log_part(disc)
    rb = disc.rules
    p = disc.space.degree
    return (lp.path == "circulant" and disc.near_k == 0 and 2 <= p <= 5 and rb.WG == 2 * p + 1
            and np.all(rb.width == rb.WG) and np.all(np.diff(rb.start) == 2)
            and disc.nodes.n == 2 * disc.space.dim)


def _assemble_into(disc: Discretization, X, scaled: bool = True):
    """Enqueue the whole assembly on the current stream (no host sync)."""
    alpha = -1.0 / (2.0 * TWO_PI) if scaled else 0.5
    if _use_v2(disc):
        return _assemble_v2(disc, X, alpha)
    skip = _ik1_skipped(disc)
    if not skip:
        _ik1_into(disc, X, accumulate=False)
    _ik2_x2_into(disc, X, accumulate=not skip, sym_alpha=alpha)
    return X


class AssemblyGraph:
    """The whole device assembly of one discretization captured once as a CUDA
    graph and replayed: one graph launch per assembly instead of ~15 kernel
    launches plus the host-side work of ``_assemble_into`` -- the step is
    launch/host-bound below N ~ 8k (C2: 0.34 ms eager for 0.06 ms of kernels).
    ``X`` is the (N, N) device output, fixed at capture; replays are
    bit-identical to eager assemblies.  The geometry flag is not checked by
    ``replay`` (call ``check`` once after the first replay)."""

    def __init__(self, disc: Discretization, X, scaled: bool = True):
        torch = _torch()
        self.disc, self.X = disc, X
        _assemble_into(disc, X, scaled)          # uploads, tables, attributes: outside capture
        torch.cuda.synchronize()
        _check_flag(_smooth(disc))
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(self.graph, stream=side):
                _assemble_into(disc, X, scaled)
        torch.cuda.current_stream().wait_stream(side)

    def replay(self):
        self.graph.replay()
        return self.X

    def check(self):
        _check_flag(_smooth(self.disc))


def assemble_matrix_device(disc: Discretization, scaled: bool = True, out=None):
    """Device-resident A = -(X + X^T)/(4 pi) (scaled) or M = (X + X^T)/2.
    Returns a torch CUDA tensor; no host synchronisation except the geometry
    flag check."""
    X = _new_square(disc) if out is None else out
    _assemble_into(disc, X, scaled)
    _check_flag(_smooth(disc))
    return X


def _gpu_local_cpus(torch):
    """CPUs on the NUMA node of the current GPU's PCIe root (sysfs local_cpulist), or
    None when unknown."""
    try:
        pr = torch.cuda.get_device_properties(torch.cuda.current_device())
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
            spec = f.read().strip()
    except (OSError, AttributeError, RuntimeError):
        return None
    cpus = set()
    for part in spec.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus or None


def pinned_host_matrix(n: int, m: int = None):
    """(n, m) float64 pinned host tensor whose pages sit on the GPU's NUMA node: the
    allocating (pinning) thread is moved onto the GPU-local CPUs for the call, so the
    device-to-host stream of the streamed host path does not cross the socket
    interconnect on multi-socket hosts (a no-op where every CPU is GPU-local)."""
    import os
    torch = _torch()
    m = n if m is None else m
    local = _gpu_local_cpus(torch)
    old = None
    if local and hasattr(os, "sched_setaffinity"):
        try:
            old = os.sched_getaffinity(0)
            use = local & old or local
            os.sched_setaffinity(0, use)
        except OSError:
            old = None
    try:
        return torch.empty((n, m), dtype=torch.float64, pin_memory=True)
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)


_COPY_STREAMS = {}


def _copy_stream(torch):
    dev = torch.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[dev]


def assemble_matrix_to_host(disc: Discretization, out=None, scaled: bool = True,
                            chunks: int = 32, work=None, devices=None):
    """A (scaled) or M into a host tensor, streaming finished row blocks to the
    host while the next ones are assembled (closed uniform meshes: tile pairs
    are processed in tile-row order, so once the pairs of tile rows < R are
    done, rows < 64 R are final).  ``out``: (N, N) float64 CPU tensor, pinned
    for full PCIe speed (allocated when None).  Other meshes assemble, then
    copy.  ``work``: optional (N, N) device buffer for the assembly (else one is
    cached on the discretization).  ``devices``: several CUDA devices assemble
    in one process, each its own share of the rows over its own PCIe link
    (``_to_host_multi``).  Returns ``out`` after the last copy."""
    torch = _torch()
    N = disc.space.dim
    if out is None:
        out = pinned_host_matrix(N)
    if devices is not None and len(devices) > 1:
        return _to_host_multi(disc, out, scaled, chunks, list(devices))
    X = work if work is not None else _dev(disc, "host_stage", lambda: _new_square(disc))
    if not _use_v2(disc) or chunks <= 1:
        _assemble_into(disc, X, scaled)
        _check_flag(_smooth(disc))
        out.copy_(X)
        return out
    alpha = -1.0 / (2.0 * TWO_PI) if scaled else 0.5
    lp, d = _logpart_dev(disc)
    sm = _smooth(disc)
    main = torch.cuda.current_stream()
    st = _lib.stream_handle(main)
    Zext = _zext_table(disc)
    x2args = (N, disc.space.degree, lp.da + 1, lp.nApad, lp.s_w.shape[1], lp.uext.shape[1],
              lp.zstride, _lib.ptr(d["uext"]), _lib.ptr(Zext), _lib.ptr(d["s_w"]), alpha, 2.0)
    T = _lib.WQ_FTILE
    nb = -(-N // T)
    start = lambda r: r * nb - r * (r - 1) // 2     # first pair of tile row r
    rows_per = max(1, -(-nb // chunks))
    cs = _copy_stream(torch)
    cs.wait_stream(main)
    done = 0
    for r0 in range(0, nb, rows_per):
        r1 = min(nb, r0 + rows_per)
        a, b = start(r0), start(r1)
        _lib.call("wq_ik1_pairs", ctypes_ref(sm["struct"]), a, b, _lib.ptr(X), X.stride(0),
                  _lib.ptr(sm["flag"]), st)
        _lib.call("wq_x2_pairs_range", *x2args, a, b, _lib.ptr(X), X.stride(0), st)
        ev = torch.cuda.Event()
        ev.record(main)
        end = min(N, r1 * T)
        cs.wait_event(ev)
        with torch.cuda.stream(cs):
            out[done:end].copy_(X[done:end], non_blocking=True)
        done = end
    cs.synchronize()
    _check_flag(sm)
    return out


def _own_row_pairs(nb: int, t0: int, t1: int) -> np.ndarray:
    """Upper-triangle tile pairs (J, I), J < t0 <= I < t1, in pair order: the
    pairs whose mirrors complete the left part of tile rows [t0, t1)."""
    if t0 == 0 or t1 <= t0:
        return np.zeros(0, np.int64)
    J = np.arange(t0, dtype=np.int64)
    first = J * nb - J * (J - 1) // 2 + (t0 - J)          # pair (J, t0)
    return (first[:, None] + np.arange(t1 - t0, dtype=np.int64)[None, :]).ravel()


def _to_host_multi(disc: Discretization, out, scaled: bool, chunks: int, devices):
    """Single-process multi-GPU host path (closed uniform meshes): the tile rows
    are split evenly over ``devices``; device d computes every tile pair that
    touches its rows -- the pairs (J, I), J < t0, whose mirrors complete the left
    part of its rows (an explicit pair list), then its own upper pairs in
    tile-row chunks -- in its own (N, N) buffer, and streams each finished row
    chunk to the shared pinned host array over its own PCIe link.  The same
    device may appear twice (two buffers on one GPU: the bit-identity test).
    Other meshes: the first device assembles, then copies."""
    torch = _torch()
    N = disc.space.dim
    if not _use_v2(disc):
        with torch.cuda.device(devices[0]):
            return assemble_matrix_to_host(disc, out=out, scaled=scaled, chunks=1)
    alpha = -1.0 / (2.0 * TWO_PI) if scaled else 0.5
    T = _lib.WQ_FTILE
    nb = -(-N // T)
    k = len(devices)
    bounds = [nb * d // k for d in range(k + 1)]
    start = lambda r: r * nb - r * (r - 1) // 2     # first pair of tile row r
    pending = []
    for slot, dev in enumerate(devices):
        t0, t1 = bounds[slot], bounds[slot + 1]
        if t1 <= t0:
            continue
        with torch.cuda.device(dev):
            lp, d = _logpart_dev(disc)
            sm = _smooth(disc)
            X = _dev(disc, ("host_multi", slot), lambda: _new_square(disc))
            plist = _dev(disc, ("host_pairs", slot, nb, t0, t1),
                         lambda: _to_dev(torch, _own_row_pairs(nb, t0, t1)))
            main = torch.cuda.current_stream()
            st = _lib.stream_handle(main)
            Zext = _zext_table(disc)
            x2args = (N, disc.space.degree, lp.da + 1, lp.nApad, lp.s_w.shape[1],
                      lp.uext.shape[1], lp.zstride, _lib.ptr(d["uext"]), _lib.ptr(Zext),
                      _lib.ptr(d["s_w"]), alpha, 2.0)
            if plist.numel():
                _lib.call("wq_ik1_pair_list", ctypes_ref(sm["struct"]), _lib.ptr(plist),
                          plist.numel(), _lib.ptr(X), X.stride(0), _lib.ptr(sm["flag"]), st)
                _lib.call("wq_x2_pair_list", *x2args, _lib.ptr(plist), plist.numel(), _lib.ptr(X),
                          X.stride(0), st)
            cs = _copy_stream(torch)
            cs.wait_stream(main)
            rows_per = max(1, -(-(t1 - t0) // max(1, chunks // k)))
            for r0 in range(t0, t1, rows_per):
                r1 = min(t1, r0 + rows_per)
                _lib.call("wq_ik1_pairs", ctypes_ref(sm["struct"]), start(r0), start(r1), _lib.ptr(X),
                          X.stride(0), _lib.ptr(sm["flag"]), st)
                _lib.call("wq_x2_pairs_range", *x2args, start(r0), start(r1), _lib.ptr(X), X.stride(0),
                          st)
                ev = torch.cuda.Event()
                ev.record(main)
                cs.wait_event(ev)
                a, b = r0 * T, min(N, r1 * T)
                with torch.cuda.stream(cs):
                    out[a:b].copy_(X[a:b], non_blocking=True)
            pending.append((dev, cs, sm))
    for dev, cs, sm in pending:
        with torch.cuda.device(dev):
            cs.synchronize()
            _check_flag(sm)
    return out


def assemble_ik1(disc: Discretization) -> np.ndarray:
    """Smooth-part Galerkin matrix IK1 = G K1 G^T (assembly.py:175-183)."""
    X = _new_square(disc)
    _ik1_into(disc, X)
    _check_flag(_smooth(disc))
    return X.cpu().numpy()


def assemble_ik2(disc: Discretization) -> np.ndarray:
    """Log-part matrix Theta C + (Theta C)^T - C^T D C (assembly.py:186-245),
    as (X2 + X2^T)/2 of the X-form."""
    X = _new_square(disc)
    if _use_v2(disc):
        _assemble_v2(disc, X, 0.5, w_ik1=0.0)
        return X.cpu().numpy()
    _ik2_x2_into(disc, X, accumulate=False, sym_alpha=0.5)
    return X.cpu().numpy()


def assemble_weighted_matrix(disc: Discretization):
    """(M, {"kernel_evals": n_quad^2}, seconds) (assembly.py:248-259); the
    seconds cover the device assembly (pair table, IK1, IK2, symmetrise)."""
    torch = _torch()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X = assemble_matrix_device(disc, scaled=False)
    torch.cuda.synchronize()
    seconds = time.perf_counter() - t0
    return X.cpu().numpy(), {"kernel_evals": disc.nodes.n ** 2}, seconds


def scale_and_symmetrize(m):
    """A = (a + a^T)/2 with a = -m/(2 pi), and the relative symmetry defect
    max|a - a^T| / max|a| (assembly.py:262-271).  Accepts a numpy array or a
    square torch CUDA tensor (returned on the device)."""
    torch = _torch()
    on_dev = hasattr(m, "is_cuda") and m.is_cuda
    X = m.to(torch.float64).contiguous().clone() if on_dev else _to_dev(torch, np.asarray(m, float))
    n = X.shape[0]
    if X.ndim != 2 or X.shape[1] != n:
        raise UsageError("scale_and_symmetrize needs a square matrix")
    stats = torch.empty(2, dtype=torch.float64, device="cuda")
    st = _lib.stream_handle()
    _lib.call("wq_absmax_defect", _lib.ptr(X), n, _lib.ptr(stats), st)
    _lib.call("wq_symmetrize", _lib.ptr(X), n, -1.0 / (2.0 * TWO_PI), st)
    mx, df = stats.cpu().numpy()
    defect = float(df / mx) if mx > 0 else 0.0
    return (X if on_dev else X.cpu().numpy()), defect


def assemble_b1_weighted(disc: Discretization, dirichlet) -> np.ndarray:
    """b1 through the regular weighted rules, one datum evaluation per node
    (assembly.py:312-319): a banded matvec on the GPU."""
    torch = _torch()
    sm = _smooth(disc)
    g = _to_dev(torch, np.asarray(dirichlet(disc.nodes.nodes), dtype=float))
    b = torch.empty(disc.space.dim, dtype=torch.float64, device="cuda")
    _lib.call("wq_b1w", ctypes_ref(sm["struct"]), _lib.ptr(g), _lib.ptr(b), _lib.stream_handle())
    return b.cpu().numpy()


def _graded_points(lo, hi, order, toward_lo, toward_hi, levels=_GRADE_LEVELS,
                   ratio=_GRADE_RATIO):
    """Composite Gauss panels shrinking toward flagged ends (assembly.py:349-378)."""
    def one_side(p_lo, p_hi, to_lo):
        h = p_hi - p_lo
        cuts = h * ratio ** np.arange(levels + 1)
        edges = np.concatenate([[0.0], cuts[::-1]])
        if to_lo:
            return np.column_stack([p_lo + edges[:-1], p_lo + edges[1:]])
        return np.column_stack([p_hi - edges[1:], p_hi - edges[:-1]])[::-1]

    if toward_lo and toward_hi:
        mid = 0.5 * (lo + hi)
        panels = np.vstack([one_side(lo, mid, True), one_side(mid, hi, False)])
    elif toward_lo:
        panels = one_side(lo, hi, True)
    elif toward_hi:
        panels = one_side(lo, hi, False)
    else:
        panels = np.array([[lo, hi]])
    x, w = np.polynomial.legendre.leggauss(order)
    half = 0.5 * (panels[:, 1] - panels[:, 0])
    mid = 0.5 * (panels[:, 0] + panels[:, 1])
    return (mid[:, None] + half[:, None] * x[None, :]).ravel(), (half[:, None] * w[None, :]).ravel()


def assemble_b1(curve, space, dirichlet, order: int = 16) -> np.ndarray:
    """b1[i] = int B_i u_D J ds by per-element Gauss, graded at open ends
    (assembly.py:287-309).  O(N) host work (not on the O(N^2) path)."""
    curve = as_curve(curve)
    space = as_basis(space)
    _check_space(curve, space)
    els = space.elements
    if space.closed:
        x, w = np.polynomial.legendre.leggauss(order)
        half = 0.5 * (els[:, 1] - els[:, 0])
        mid = 0.5 * (els[:, 0] + els[:, 1])
        pts = (mid[:, None] + half[:, None] * x[None, :]).ravel()
        wts = (half[:, None] * w[None, :]).ravel()
    else:
        last = len(els) - 1
        pp = [_graded_points(lo, hi, order, e == 0, e == last) for e, (lo, hi) in enumerate(els)]
        pts = np.concatenate([p for p, _ in pp])
        wts = np.concatenate([w for _, w in pp])
    vals = np.asarray(dirichlet(pts), dtype=float)
    bv, bc = active_values(space, pts)
    jac = np.linalg.norm(curve.spline(1)(np.clip(pts, curve.basis.a, curve.basis.b)), axis=-1)
    out = np.zeros(space.dim)
    np.add.at(out, bc.ravel(), (bv * (wts * jac * vals)[:, None]).ravel())
    return out


def assemble_b2(curve, space, dirichlet, order: int = 16) -> np.ndarray:
    """b2[i] = 1/(2 pi) int B_i J [int Kbar(s,t) u_D(t) dt] ds by per-element
    Gauss on both integrals (assembly.py:322-343).  The (M x M) Kbar grid,
    M = order * n_el, is evaluated on the GPU (wq_b2_inner) and never stored;
    the diagonal uses the C^2 curvature limit (geometry.py:269-279)."""
    torch = _torch()
    curve = as_curve(curve)
    space = as_basis(space)
    _check_space(curve, space)
    if not curve.is_c2():
        raise GeometryError("double-layer right-hand side needs a C^2 curve")
    els = space.elements
    x, w = np.polynomial.legendre.leggauss(order)
    half = 0.5 * (els[:, 1] - els[:, 0])
    mid = 0.5 * (els[:, 0] + els[:, 1])
    pts = (mid[:, None] + half[:, None] * x[None, :]).ravel()
    wts = (half[:, None] * w[None, :]).ravel()
    b = curve.basis
    cp = np.clip(pts, b.a, b.b)
    f = curve.spline(0)(cp)
    d1 = curve.spline(1)(cp)
    d2 = curve.spline(2)(cp)
    kdiag = 0.5 * (d1[:, 1] * d2[:, 0] - d1[:, 0] * d2[:, 1]) / np.sum(d1 ** 2, axis=-1)
    wg = wts * np.asarray(dirichlet(pts), dtype=float)
    dev = [_to_dev(torch, a) for a in (f[:, 0], f[:, 1], d1[:, 0], d1[:, 1], wg, kdiag)]
    inner = torch.empty(len(pts), dtype=torch.float64, device="cuda")
    _lib.call("wq_b2_inner", len(pts), *[_lib.ptr(t) for t in dev], _lib.ptr(inner),
              _lib.stream_handle())
    inner = inner.cpu().numpy()
    jac = np.linalg.norm(d1, axis=-1)
    bv, bc = active_values(space, pts)
    out = np.zeros(space.dim)
    np.add.at(out, bc.ravel(), (bv * (wts * jac * inner)[:, None]).ravel())
    return out / TWO_PI
