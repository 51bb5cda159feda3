"""CPU: the O(N) host precompute of the product against the reference's
outputs, and a numpy execution of the exact GPU dataflow (same host arrays,
same index conventions as the kernels) against the reference matrix."""

import numpy as np
import pytest

import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, precompute as PC
from paper_1703_10016_b200.errors import ConstructionError, UsageError
from oracle import wq_oracle as O
from _cases import golden_names, load, product_objects, rel

FULL = [n for n in golden_names() if "G" in load(n)[0]]


@pytest.mark.parametrize("name", golden_names())
def test_nodes_match_reference(name):
    z, meta = load(name)
    curve, space = product_objects(meta)
    disc = W.build_discretization(curve, space, meta["nref"])
    assert np.array_equal(disc.nodes.nodes, z["nodes"])
    assert np.array_equal(disc.J_nodes, z["J_nodes"])  # same scipy evaluation
    assert disc.nodes.n == meta["nq"]


@pytest.mark.parametrize("name", FULL)
def test_rule_band_matches_reference_G(name):
    z, meta = load(name)
    curve, space = product_objects(meta)
    disc = W.build_discretization(curve, space, meta["nref"])
    G = disc.G
    assert np.array_equal(G != 0, z["G"] != 0)
    # min-norm solver differences live in the exactness null space
    # (SURVEY sec.7 iii: <= 8.8e-11 at p=5, effect on IK1 <= 2e-15)
    tol = {2: 1e-13, 3: 1e-12, 4: 1e-10, 5: 1e-9}[space.degree]
    assert rel(G, z["G"]) <= tol


def _emulate_gpu_dataflow(disc):
    """numpy rendition of wq_ik1 + wq_pair_table + wq_circ_tables +
    wq_ik2_circ / general path + wq_symmetrize on the product's arrays."""
    N = disc.space.dim
    nodes = disc.nodes.nodes
    ocurve = O.Curve(disc.curve.basis, disc.curve.control_points)
    X = disc.G @ O.k1_grid(ocurve, nodes, nodes) @ disc.G.T
    lp = AS._log_part(disc)
    n = lp.n_el
    m2, _ = O.uniform_pair_moments(O.as_basis(disc.refined.basis), lp.da)
    if lp.path == "circulant":
        nB = lp.db + 1
        Z = sum(np.roll(m2, b, axis=0) @ lp.v0[:, b] for b in range(nB))
        dd = sum(np.roll(Z[:, :nB], -a, axis=0) @ lp.v0[:nB, a] for a in range(nB))
        K = (len(lp.hinv_taps) - 1) // 2
        corr = lambda arr: sum(np.roll(arr, -k, axis=0) * lp.hinv_taps[K + k] for k in range(-K, K + 1))
        Zp, ff = corr(Z), corr(corr(dd))
        m = np.arange(n)
        Phi = np.zeros((n, N))
        for i in range(N):
            for a in range(lp.U.shape[1]):
                Phi[:, i] += 2 * Zp[np.mod(m - lp.e_start[i] - a, n)] @ lp.U[i, a]
            for t in range(lp.s_w.shape[1]):
                Phi[:, i] -= lp.s_w[i, t] * ff[np.mod(m - lp.s_start[i] - t, n)]
        X2 = np.zeros((N, N))
        for j in range(N):
            for t in range(lp.s_w.shape[1]):
                X2[:, j] += lp.s_w[j, t] * Phi[(lp.s_start[j] + t) % n]
        X = X + X2
    else:
        import scipy.linalg as sl
        NE = disc.refined.basis.dim
        gap = (lambda e, f: (f - e) % n) if disc.closed else (lambda e, f: f - e + n - 1)
        thT = np.zeros((NE, N))
        D = np.zeros((NE, NE))
        for l in range(NE):
            for f, b in zip(lp.v_el[l], lp.v_loc[l]):
                if f < 0:
                    continue
                for i in range(N):
                    for e, a in zip(lp.u_el[i], lp.u_loc[i]):
                        if e >= 0:
                            thT[l, i] += lp.u[e][:, a] @ m2[gap(e, f)] @ lp.v[f][:, b]
                for mm in range(NE):
                    for e, a in zip(lp.v_el[mm], lp.v_loc[mm]):
                        if e >= 0:
                            D[mm, l] += lp.v[e][:, a] @ m2[gap(e, f)][: lp.db + 1] @ lp.v[f][:, b]
        L = np.zeros((NE, NE))
        m = lp.Lb.shape[0]
        for j in range(lp.bw + 1):
            L[np.arange(j, m), np.arange(0, m - j)] = lp.Lb[j:, j]
        if lp.L21 is not None:   # closed mesh: arrow-shaped factor
            L[m:, :m] = lp.L21
            L[m:, m:] = lp.L22
        hinv = lambda Y: sl.solve_triangular(L.T, sl.solve_triangular(L, Y, lower=True))
        F = hinv(hinv(D).T)
        Phi = 2 * hinv(thT)
        for i in range(N):
            for t in range(lp.s_w.shape[1]):
                Phi[:, i] -= F[:, (lp.s_start[i] + t) % NE] * lp.s_w[i, t]
        X2T = np.zeros((N, N))
        for j in range(N):
            for t in range(lp.s_w.shape[1]):
                X2T[j] += lp.s_w[j, t] * Phi[(lp.s_start[j] + t) % NE]
        X = X + X2T
    return -(X + X.T) / (4 * np.pi)


@pytest.mark.parametrize("name", ["ell_p3_n32", "ell_p2_n64", "ell_p5_n64", "star_p4_n128",
                                  "c1_slit_p2_n64", "slit_p4_n24_dbl", "parabola_p3_n16",
                                  "slit_p5_n24", "closed_smooth_p3_n24", "ell_p3_n32_nref2",
                                  "slit_p2_n16_nref2"])
def test_gpu_dataflow_in_numpy_matches_reference(name):
    z, meta = load(name)
    curve, space = product_objects(meta)
    disc = W.build_discretization(curve, space, meta["nref"])
    assert rel(_emulate_gpu_dataflow(disc), z["A"]) <= 5e-14


def test_k1_distance_modes():
    z, meta = load("ell_p3_n64")
    curve, space = product_objects(meta)
    disc = W.build_discretization(curve, space, 1)
    assert disc.k1_mode == 0 and disc.invp2 is not None   # uniform binary nodes -> gap table
    x = np.abs(disc.nodes.nodes - disc.nodes.nodes[0])
    L = curve.length
    p = (L / np.pi) * np.abs(np.sin(np.pi * x / L))
    assert np.array_equal(disc.invp2[1:], 1.0 / (p[1:] * p[1:]))
    z, meta = load("c1_slit_p2_n64")
    curve, space = product_objects(meta)
    assert W.build_discretization(curve, space, 1).k1_mode == 1  # open: graded end nodes


def test_circulant_detection_and_taps():
    curve, space = product_objects(load("ell_p3_n128")[1])
    lp = AS._log_part(W.build_discretization(curve, space, 1))
    assert lp.path == "circulant"
    K = (len(lp.hinv_taps) - 1) // 2
    assert np.allclose(lp.hinv_taps, lp.hinv_taps[::-1], rtol=0, atol=1e-15 * abs(lp.hinv_taps[K]))
    if 2 * K + 1 < 128:
        assert abs(lp.hinv_taps[0]) <= 1e-18 * abs(lp.hinv_taps[K])


def test_errors_mirror_reference():
    curve, _ = product_objects(load("ell_p3_n64")[1])
    with pytest.raises(UsageError):
        W.build_discretization(curve, W.make_open_basis(3, np.linspace(0, 1, 9)), 1)
    slit = W.load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
    graded = W.make_open_basis(2, np.array([-1, -0.9, -0.5, 0.0, 0.5, 0.9, 1.0]))
    disc = W.build_discretization(slit, graded, 1)
    # the reference raises here (quadrature.py:489-491); graded meshes take the
    # per-pair route instead (config 5), the uniform-width helper still raises
    with pytest.raises(ConstructionError, match="uniform element mesh"):
        PC.uniform_width(disc.refined.basis)
    lp = AS._log_part(disc)
    assert lp.graded and lp.path == "general" and lp.h is None


def _near_brute(fine):
    els = fine.elements
    h = els[:, 1] - els[:, 0]
    mid = 0.5 * (els[:, 0] + els[:, 1])
    delta = mid[:, None] - mid[None, :]
    if fine.closed:
        delta = delta - fine.length * np.round(delta / fine.length)
    sep = np.abs(delta) - 0.5 * (h[:, None] + h[None, :])
    return sep <= PC.NEAR_TOUCH * np.maximum(h[:, None], h[None, :])


@pytest.mark.parametrize("closed", [False, True])
@pytest.mark.parametrize("n", [3, 7, 40])
def test_element_pair_geometry_matches_predicate(closed, n):
    rng = np.random.default_rng(n)
    c = np.cumsum(rng.normal(0.0, 0.5, n))          # widths drifting over decades
    if closed:                                      # ... and matching across the seam
        c -= np.arange(n) / max(n - 1, 1) * (c[-1] - c[0])
    w = np.exp(c)
    bp = np.concatenate([[0.0], np.cumsum(w)])
    bp = bp / bp[-1]
    space = W.make_cyclic_basis(2, bp) if closed else W.make_open_basis(2, bp)
    fine = W.refine_uniform(space, 1).basis
    h, mid, lo, cnt = PC.element_pair_geometry(fine)
    near = _near_brute(fine)
    got = np.zeros_like(near)
    for e in range(n):
        got[e, np.mod(lo[e] + np.arange(cnt[e]), n)] = True
    # ranges are contiguous covers of the near set (gaps inside would take the
    # closed form, which is exact for any offset); here they coincide
    assert np.array_equal(got, near)
    assert np.all(cnt >= 1) and np.all(cnt <= n)


def test_touching_width_ratio_limit():
    bp = np.array([0.0, 0.01, 0.1, 0.5, 1.0])     # 0.01 next to 0.09: ratio 9
    with pytest.raises(ConstructionError, match="width ratio"):
        PC.element_pair_geometry(W.make_open_basis(2, bp))
    x, w = PC.log_gauss_unit(PC.TOUCH_LOG)          # weight -ln x on (0, 1)
    k = np.arange(2 * PC.TOUCH_LOG)
    assert np.abs((w[None, :] * x[None, :] ** k[:, None]).sum(1) * (k + 1.0) ** 2 - 1).max() < 1e-14


def test_config5_mesh_reading():
    space = O.config5_space()
    assert space.dim == 20418          # 16384 elements + 4030 doubled knots (default_rng(0))
    h = np.diff(space.breakpoints)
    assert h.min() / h.max() == pytest.approx(0.9 ** 60, rel=1e-9)


def test_precompute_is_linear_time():
    import time
    space = W.make_cyclic_basis(3, np.linspace(0, 1, 8193))
    t0 = time.perf_counter()
    fine = W.refine_uniform(space, 1).basis
    nodes = PC.build_nodes(fine)
    rb = PC.regular_rule_band(space, fine, nodes)
    assert time.perf_counter() - t0 < 30.0
    assert rb.WG == 7 and np.ptp(rb.weights, axis=0).max() < 1e-15


def test_graded_gather_dataflow_in_numpy():
    """numpy rendition of the graded-mesh route (wq_gen_pair_blocks per chunk
    of outer elements + wq_gen_gather_theta / wq_gen_gather_d with the host's
    incidence arrays and chunk index ranges) against the restatement's Theta, D."""
    for closed in (False, True):
        rng = np.random.default_rng(11)
        n = 24
        w = np.exp(0.5 * rng.normal(size=n))
        bp = np.concatenate([[0.0], np.cumsum(w)]) / w.sum()
        if closed:
            th = 2 * np.pi * np.arange(16) / 16
            curve = W.load_curve({"degree": 3, "closed": True,
                                  "breakpoints": np.linspace(0, 1, 17).tolist(),
                                  "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})
            space = W.make_cyclic_basis(2, bp)
        else:
            curve = W.load_curve({"degree": 1, "knots": [0, 0, 1, 1], "control_points": [[-1, 0], [1, 0]]})
            space = W.make_open_basis(3, bp, np.where(rng.random(n - 1) < 0.3, 2, 1))
        disc = W.build_discretization(curve, space, 1)
        lp = AS._log_part(disc)
        assert lp.graded
        N, NE = space.dim, disc.refined.basis.dim
        fine = disc.refined.basis
        delta_all = lp.elm[:, None] - lp.elm[None, :]
        if closed:
            delta_all = delta_all - fine.length * np.round(delta_all / fine.length)
        thT = np.zeros((NE, N))
        D = np.zeros((NE, NE))
        chunk = 5
        for e0 in range(0, n, chunk):
            e1 = min(n, e0 + chunk)
            es = np.arange(e0, e1)
            he = np.repeat(lp.elh[es], n)
            hf = np.tile(lp.elh, len(es))
            m2 = O.pair_moments_general(lp.da, lp.db, he, hf, delta_all[es].ravel(),
                                        closed_period=fine.length if closed else None)
            m2 = m2.reshape(len(es), n, lp.da + 1, lp.db + 1)
            wt = np.einsum("eap,efab,fbq->efpq", lp.u[es], m2, lp.v)
            wd = np.einsum("eap,efab,fbq->efpq", lp.v[es], m2[:, :, : lp.db + 1], lp.v)
            uc, vc = lp.ucols[e0:e1], lp.vcols[e0:e1]
            for i in range(int(uc.min()), int(uc.max()) + 1):
                for e, a in zip(lp.u_el[i], lp.u_loc[i]):
                    if e0 <= e < e1:
                        for l in range(NE):
                            for f, b in zip(lp.v_el[l], lp.v_loc[l]):
                                if f >= 0:
                                    thT[l, i] += wt[e - e0, f, a, b]
            for l in range(int(vc.min()), int(vc.max()) + 1):
                for e, a in zip(lp.v_el[l], lp.v_loc[l]):
                    if e0 <= e < e1:
                        for m in range(NE):
                            for f, b in zip(lp.v_el[m], lp.v_loc[m]):
                                if f >= 0:
                                    D[l, m] += wd[e - e0, f, a, b]
        od = O.build_discretization(O.Curve(curve.basis, curve.control_points),
                                    O.Basis(space.degree, space.knots, space.closed), 1)
        theta, dmm, _ = O.ik2_ingredients_general(od)
        assert rel(thT.T, theta) <= 1e-13
        assert rel(D, dmm) <= 1e-13


def test_regular_rules_list_like_reference():
    """disc.regular_rules is the reference's list of WeightedRule
    (quadrature.py:150-176): stacking it as rules_matrix does, times J, gives G;
    singular_rules raises a clear UsageError (not built)."""
    from paper_1703_10016_b200.errors import UsageError
    z, meta = load("slit_p4_n24_dbl")
    curve, space = product_objects(meta)
    disc = W.build_discretization(curve, space, 1)
    rules = disc.regular_rules
    assert len(rules) == space.dim and rules[3].tag == ("basis", 3)
    dense = np.zeros((len(rules), disc.nodes.n))
    for k, r in enumerate(rules):
        dense[k, r.idx] = r.weights
    assert np.array_equal(dense * disc.J_nodes[None, :], disc.G)
    g = np.cos(disc.nodes.nodes)
    assert abs(rules[5].apply(g) - rules[5].full_weights(disc.nodes.n) @ g) <= 1e-15
    with pytest.raises(UsageError):
        disc.singular_rules


def test_inverse_decay_rows_bounds_dense_inverse():
    """precompute.inverse_decay_rows (warm-up of the segmented device solves)
    bounds where the columns of L^{-1} and L^{-T} fall below 1e-20 of their peak,
    against dense inverses of the fit factor of a config-5 reading."""
    from oracle import wq_oracle as O
    from paper_1703_10016_b200 import assembly as AS, precompute as PC
    sp = O.config5_space(n_el=512)
    curve = W.load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
    disc = W.build_discretization(curve, W.BasisSpec(sp.degree, sp.knots, False), 1)
    lp = AS._log_part(disc)
    k = PC.inverse_decay_rows(lp.Lb, lp.bw)
    assert 0 < k < 200
    m = lp.Lb.shape[0]
    L = np.zeros((m, m))
    for j in range(lp.bw + 1):
        L[np.arange(j, m), np.arange(m - j)] = lp.Lb[j:, j]
    Li = np.linalg.inv(L)
    for c in range(0, m - k, 37):
        col = np.abs(Li[c:, c])
        assert np.all(col[k:] < 1e-19 * col.max())


def test_end_node_fix_opt_in():
    """A repeated knot next to an open end element: the reference drops the
    extra end-element nodes (quadrature.py:106-108) and then raises on the
    rank-deficient last rule (quadrature.py:528-531) -- the default here does
    the same; the opt-in end_node_fix keeps them and the rules are exact."""
    from oracle import wq_oracle as O
    from paper_1703_10016_b200.errors import ConstructionError
    curve = W.load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
    sp = O.config5_space(n_el=64, growth_elems=12)
    assert sp.multiplicities[-2] == 2
    space = W.BasisSpec(sp.degree, sp.knots, False)
    with pytest.raises(ConstructionError):
        W.build_discretization(curve, space, 1)
    disc = W.build_discretization(curve, space, 1, end_node_fix=True)
    n_default = len(O.build_nodes(sp))
    assert disc.nodes.n == n_default + 1
    od = O.build_discretization(O.Curve(curve.basis, curve.control_points), sp, 1, end_fix=True)
    assert np.array_equal(od.nodes, disc.nodes.nodes)
    assert np.abs(disc.G - od.G).max() <= 1e-9 * np.abs(od.G).max()
