"""Pins of the oracle's STree + vMF guide (§5.5-5.6).

CPU only.  Expected values come from the mathematics the paper fixes, not
from the oracle: the vMF law of Eq. 12 (closed-form mean cosine, CDF, the
uniform limit), the spatial meaning of the tree (every sample lies in the leaf
its own configuration reaches; leaves respect the sqrt|S| threshold; eps = 0
reduces to a partition), brute-force nearest neighbours for kappa = sigma^-2,
and the mixture probabilities of Eqs. 10, 11 and 13 recomputed from the raw
sample weights.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12818_b200 import workloads as W


def _records(n=6000, seed=1, **kw):
    r = W.synthetic_guide_samples(n, seed, **kw)
    return np.frombuffer(r.tobytes(), O.GSAMPLE).copy()


def _key(r):
    return np.concatenate([r["xD"], r["xL"]], axis=1) + np.float32(0.0)


def _descend(G, p):
    ref = G["root_ref"]
    depth = 0
    while ref >= 0:
        nd = G["nodes"][ref]
        ref = int(nd["child"][0] if p[nd["axis"]] < nd["split"] else nd["child"][1])
        depth += 1
    return ~ref, depth


# ---------------------------------------------------------------------------
# vMF sampling (Eq. 12): v(w; mu, kappa) = kappa / (4 pi sinh kappa) e^{kappa mu.w}
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("kappa", [0.5, 4.0, 60.0, 5000.0])
def test_vmf_mean_cosine_and_cdf(kappa):
    rng = np.random.default_rng(7)
    mu = rng.normal(size=3)
    mu = (mu / np.linalg.norm(mu)).astype(np.float32)
    n = 4000
    u = (np.arange(n) + rng.random(n)) / n           # stratified in u1 (cos theta)
    u = np.floor(u * 2**24) / 2**24
    v = np.floor(rng.random(n) * 2**24) / 2**24
    W_ = np.array([O.vmf_sample(mu, kappa, a, b) for a, b in zip(u, v)], np.float64)
    assert np.allclose(np.linalg.norm(W_, axis=1), 1.0, atol=2e-6)
    c = W_ @ mu.astype(np.float64)
    # E[mu.w] = coth(kappa) - 1/kappa (closed form of Eq. 12); stratified u1 -> tiny error
    expect = 1.0 / np.tanh(kappa) - 1.0 / kappa
    assert abs((1.0 - c.mean()) - (1.0 - expect)) < 0.01 * (1.0 - expect), (c.mean(), expect)
    # CDF F(c) = (e^{kappa c} - e^{-kappa}) / (2 sinh kappa) = e^{kappa (c-1)} (1 - e^{-kappa (c+1)}) / (1 - e^{-2 kappa})
    cs = np.sort(c)
    F = np.exp(kappa * (cs - 1.0)) * (-np.expm1(-kappa * (cs + 1.0))) / (-np.expm1(-2.0 * kappa))
    ks = np.max(np.abs(F - (np.arange(n) + 0.5) / n))
    assert ks < 2.0 / n + kappa * 1.2e-7, ks
    # azimuth uniform: the tangential part has zero mean
    t = W_ - np.outer(c, mu)
    assert np.abs(t.mean(0)).max() < 4.0 * np.sqrt((1 - (c**2).mean()) / n) + 1e-6


def test_vmf_small_kappa_is_uniform_sphere():
    rng = np.random.default_rng(3)
    mu = np.array([0.0, 1.0, 0.0], np.float32)
    n = 6000
    W_ = np.array([O.vmf_sample(mu, 1e-3, np.floor(a * 2**24) / 2**24, np.floor(b * 2**24) / 2**24)
                   for a, b in rng.random((n, 2))])
    # uniform on S^2: E[w] = 0, E[w_y^2] = 1/3
    assert np.abs(W_.mean(0)).max() < 4.0 / np.sqrt(3 * n)
    assert abs((W_[:, 1] ** 2).mean() - 1.0 / 3.0) < 4.0 * np.sqrt(4.0 / 45.0 / n)


# ---------------------------------------------------------------------------
# STree: spatial meaning, threshold, overlap
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def built():
    r = _records()
    return r, O.stree_build(r)


def test_stree_counts_and_threshold(built):
    r, G = built
    valid = (r["w"] > 0) & (r["type"] >= 0)
    assert G["n_valid"] == valid.sum()
    assert G["thr"] == int(np.floor(np.sqrt(valid.sum())))        # threshold sqrt|S| (c = 1)
    assert G["n_leaves"] == G["n_nodes"] + 1                       # full binary tree
    # every leaf below the threshold unless it sits at the depth cap
    for l in range(G["n_leaves"]):
        if G["leaf_count"][l] > G["thr"]:
            pytest.fail(f"leaf {l} holds {G['leaf_count'][l]} > thr")
    # only samples in leaves
    ids = G["leaf_ids"]
    assert valid[ids].all()


def test_stree_every_sample_in_its_own_leaf(built):
    r, G = built
    K = _key(r)
    ids = G["leaf_ids"]
    leaf_of = np.repeat(np.arange(G["n_leaves"]), G["leaf_count"])
    member = set(zip(leaf_of.tolist(), ids.tolist()))
    for i in np.nonzero((r["w"] > 0) & (r["type"] >= 0))[0]:
        leaf, _ = _descend(G, K[i])
        assert (leaf, int(i)) in member, i


def test_stree_copies_are_near_the_leaf(built):
    """Overlap copies (P:523 footnote) stay within half a child width of the leaf's box along each axis."""
    r, G = built
    K = _key(r)
    valid = (r["w"] > 0) & (r["type"] >= 0)
    lo0, hi0 = K[valid].min(0), K[valid].max(0)
    # leaf boxes by walking the tree
    boxes = {}
    stack = [(G["root_ref"], lo0.copy(), hi0.copy())]
    while stack:
        ref, lo, hi = stack.pop()
        if ref < 0:
            boxes[~ref] = (lo, hi)
            continue
        nd = G["nodes"][ref]
        a, c = int(nd["axis"]), np.float32(nd["split"])
        l2, h2 = lo.copy(), hi.copy()
        h2[a] = c
        stack.append((int(nd["child"][0]), lo.copy(), h2))
        l2[a] = c
        stack.append((int(nd["child"][1]), l2, hi.copy()))
    start = 0
    copies = 0
    for l in range(G["n_leaves"]):
        cnt = G["leaf_count"][l]
        ids = G["leaf_ids"][start:start + cnt]
        start += cnt
        lo, hi = boxes[l]
        P = K[ids].astype(np.float64)
        w = (hi - lo).astype(np.float64)
        out = np.maximum(lo - P, P - hi)
        assert (out <= 0.5 * w + 1e-6).all()
        copies += int((out > 0).any(axis=1).sum())
    assert copies > 0   # the overlap is in effect


def test_stree_eps_zero_is_a_partition():
    """eps = 0: no copies, every sample in exactly one leaf (the plain kd-tree special case)."""
    r = _records(3000, seed=5)
    G = O.stree_build(r, eps=0.0)
    ids = np.sort(G["leaf_ids"])
    assert np.array_equal(ids, np.nonzero((r["w"] > 0) & (r["type"] >= 0))[0])


def test_stree_huge_threshold_is_one_leaf():
    r = _records(2000, seed=6)
    G = O.stree_build(r, c_thr=1e6)
    assert G["n_nodes"] == 0 and G["n_leaves"] == 1 and G["root_ref"] == ~0
    assert np.array_equal(G["leaf_ids"], np.nonzero((r["w"] > 0) & (r["type"] >= 0))[0])


def test_stree_empty_sample_set():
    r = _records(500, seed=7)
    r["w"] = 0.0
    G = O.stree_build(r)
    assert G["n_leaves"] == 1 and G["n_lobes"] == 0
    # no learned energy: the length table is the initializer's P_0 alone
    npf = G["n_prefix"][0].astype(np.int64)
    assert np.array_equal(np.diff(np.concatenate([[0], npf])), [20, 20, 20, 20, 20, 19])
    assert (G["type_prefix"][0] == 0).all()


# ---------------------------------------------------------------------------
# Per-leaf distributions (Eqs. 10-13) and the vMF footprint
# ---------------------------------------------------------------------------
def test_kappa_is_inverse_square_nearest_direction(built):
    r, G = built
    lobes = G["lobe_sample"]
    for l in range(0, G["n_leaves"], 7):
        for t in range(126):
            a, b = G["grp_off"][l, t], G["grp_off"][l, t + 1]
            if b - a < 2:
                continue
            om = r["omega"][lobes[a:b]].astype(np.float64)
            d2 = ((om[:, None, :] - om[None, :, :]) ** 2).sum(-1)
            np.fill_diagonal(d2, np.inf)
            kap = 1.0 / d2.min(1)                      # Eq. 12, unclamped (the default)
            assert np.allclose(G["lobe_mu"][a:b, 3], kap, rtol=2e-4), (l, t)
            assert np.array_equal(G["lobe_mu"][a:b, :3], r["omega"][lobes[a:b]])
            assert (r["type"][lobes[a:b]] == t).all()


def test_leaf_tables_are_the_defensive_mixtures(built):
    """P(n) = 1/2 P_0(n) + 1/2 P_e(n) (Eqs. 10, 13), P_e(tau|n) (Eq. 11), lobe ~ w_i,
    each within the 2^-20 quantization of the integer tables."""
    r, G = built
    P0 = np.array([20, 20, 20, 20, 20, 19], np.float64) / 119.0
    start = 0
    for l in range(G["n_leaves"]):
        cnt = G["leaf_count"][l]
        ids = G["leaf_ids"][start:start + cnt]
        start += cnt
        w = r["w"][ids].astype(np.float64)
        ty = r["type"][ids]
        ln = np.floor(np.log2(ty + 2)).astype(int)       # type = 2^n - 2 + tau
        En = np.array([w[ln == n].sum() for n in range(1, 7)])
        if En.sum() == 0:
            continue
        npf = G["n_prefix"][l].astype(np.float64)
        Pn = np.diff(np.concatenate([[0.0], npf])) / npf[-1]
        assert np.allclose(Pn, 0.5 * P0 + 0.5 * En / En.sum(), atol=4e-6 * 6), l
        for n in range(1, 7):
            g0, gn = (1 << n) - 2, 1 << n
            Et = np.array([w[ty == g0 + m].sum() for m in range(gn)])
            tp = G["type_prefix"][l, g0:g0 + gn].astype(np.float64)
            if Et.sum() == 0:
                assert (tp == 0).all()
                continue
            Pt = np.diff(np.concatenate([[0.0], tp])) / tp[-1]
            assert np.allclose(Pt, Et / Et.sum(), atol=gn * 2e-6), (l, n)
        for t in np.unique(ty)[:4]:
            a, b = G["grp_off"][l, t], G["grp_off"][l, t + 1]
            lp = G["lobe_prefix"][a:b].astype(np.float64)
            pl = np.diff(np.concatenate([[0.0], lp])) / lp[-1]
            wl = r["w"][G["lobe_sample"][a:b]].astype(np.float64)
            assert np.allclose(pl, wl / wl.sum(), atol=(b - a) * 2e-6), (l, t)


def test_seed_mode4_draws_from_the_leaf_mixture():
    """Seeds of mode 4 on the configs[4] scene: the leaf is the one of (x_D, x_L); about half the
    draws are learned (alpha = 1/2, Eq. 13); learned directions sit in the lobes' vMF footprints."""
    w = W.config4(n_side=24, grid_n=16)
    sc = O.OracleScene(w)
    r = _records(4000, seed=11)
    G = O.stree_build(r)
    sc.set_stree(G)
    learned = 0
    near = 0
    n = 400
    for i in range(n):
        s = sc.seed_ex(i)
        assert s["ok"]
        if s["learned"]:
            learned += 1
            b = s["bin"]
            mu = G["lobe_mu"][b]
            xd = w.xD[i]
            d = s["target"].astype(np.float64) - xd
            d /= np.linalg.norm(d)
            near += float(d @ mu[:3]) >= 1.0 - 9.0 / mu[3] - 1e-6   # P(mu.w < 1 - 9/kappa) <= e^-9
            assert (s["tau"] + (1 << s["n"]) - 2) == r["type"][G["lobe_sample"][b]]
    assert 0.3 * n < learned < 0.7 * n
    assert near >= learned - 2


# ---------------------------------------------------------------------------
# glossy separator product weighting (Eq. 14; R35)
# ---------------------------------------------------------------------------
def _rho(wv, om, alpha):
    """rho via the oracle's recorder: one receiver at the origin (normal +y), walks towards om."""
    n = om.shape[0]
    xD = np.zeros((1, 3), np.float32)
    rec = O.record_samples(xD, n, np.zeros(n, np.int32), np.ones(n, np.float32), om.astype(np.float32),
                           np.ones(n, np.int32), np.zeros(n, np.uint32), np.zeros((n, 3), np.float32),
                           wv=np.asarray([wv], np.float32), nD=np.asarray([[0, 1, 0]], np.float32), alpha=alpha)
    return rec["w"].astype(np.float64)


@pytest.mark.parametrize("alpha", [0.05, 0.1])
def test_ggx_separator_lobe_normalised_at_normal_incidence(alpha):
    """int rho(n, l) cos_l dl = int D(h) (n.h) dh over the h whose reflection stays above the
    surface (theta_h <= 45 deg): the GGX mass there, 1 / (1 + alpha^2) in closed form."""
    m, mp = 8000, 8                              # midpoint rule in (cos^2 theta_l, phi); the lobe is
    u = (np.arange(m) + 0.5) / m                 # symmetric in phi at normal incidence
    ct = np.sqrt(u)                              # cos theta, area element d(omega) = d(ct^2)/2 dphi
    ph = 2 * np.pi * (np.arange(mp) + 0.5) / mp
    CT, PH = np.meshgrid(ct, ph, indexing="ij")
    ST = np.sqrt(1 - CT ** 2)
    om = np.stack([ST * np.cos(PH), CT, ST * np.sin(PH)], -1).reshape(-1, 3)
    r = _rho([0.0, 1.0, 0.0], om, alpha)
    cosl = om[:, 1]
    integral = (r * cosl / cosl).sum() * (0.5 / m) * (2 * np.pi / mp)  # rho cos_l d(omega) = rho du/2 dphi
    assert integral == pytest.approx(1.0 / (1.0 + alpha * alpha), abs=2e-3)


def test_ggx_separator_reciprocal_and_one_sided():
    rng = np.random.default_rng(2)
    v = rng.normal(size=(200, 3)); v[:, 1] = np.abs(v[:, 1]); v /= np.linalg.norm(v, axis=1, keepdims=True)
    l = rng.normal(size=(200, 3)); l[:, 1] = np.abs(l[:, 1]); l /= np.linalg.norm(l, axis=1, keepdims=True)
    a = np.array([_rho(v[i], l[i:i + 1], 0.3)[0] for i in range(50)])
    b = np.array([_rho(l[i], v[i:i + 1], 0.3)[0] for i in range(50)])
    assert np.allclose(a, b, rtol=2e-6)                                  # rho(v, l) = rho(l, v)
    below = l[:5] * np.array([1, -1, 1])
    assert (_rho(v[0], below, 0.3) == 0).all()                          # no weight below the separator


# ---------------------------------------------------------------------------
# Selective activation (reading R36)
# ---------------------------------------------------------------------------
def _leaf_boxes(G, K, valid):
    """Leaf boxes from the split planes (left: x < c, right: x >= c), root = the data box."""
    lo0, hi0 = K[valid].min(0), K[valid].max(0)
    boxes = {}
    stack = [(G["root_ref"], lo0.copy(), hi0.copy(), np.zeros(6, bool))]
    while stack:
        ref, lo, hi, cut = stack.pop()          # cut[a]: hi[a] is a split plane (strict <)
        if ref < 0:
            boxes[~ref] = (lo, hi, cut)
            continue
        nd = G["nodes"][ref]
        a, c = int(nd["axis"]), np.float32(nd["split"])
        h2, c2 = hi.copy(), cut.copy()
        h2[a], c2[a] = c, True
        stack.append((int(nd["child"][0]), lo.copy(), h2, c2))
        l2 = lo.copy()
        l2[a] = c
        stack.append((int(nd["child"][1]), l2, hi.copy(), cut.copy()))
    return boxes


def _inside(P, box):
    lo, hi, cut = box
    return np.all(P >= lo, axis=-1) & np.all(np.where(cut, P < hi, P <= hi), axis=-1)


@pytest.mark.parametrize("eps", [0.1, 0.0])
def test_leaf_own_samples_are_the_leaf_list_without_copies(eps):
    """P:606 "samples (excluding those used for filtering)": a leaf's own samples are the
    members of its list that lie inside its box (the rest are the overlap copies of P:523);
    they partition S, and with eps = 0 (no copies) they are the whole list."""
    r = _records(8000, seed=3)
    G = O.stree_build(r, eps=eps)
    K = _key(r)
    valid = (r["w"] > 0) & (r["type"] >= 0)
    boxes = _leaf_boxes(G, K, valid)
    start = 0
    own = np.zeros(G["n_leaves"], np.int64)
    for l in range(G["n_leaves"]):
        cnt = G["leaf_count"][l]
        ids = G["leaf_ids"][start:start + cnt]
        start += cnt
        own[l] = int(_inside(K[ids], boxes[l]).sum())
    assert np.array_equal(G["leaf_own"], own)
    assert own.sum() == valid.sum()                    # every sample is own in exactly one leaf
    if eps == 0.0:
        assert np.array_equal(own, G["leaf_count"])
    else:
        assert (own < G["leaf_count"]).any()           # copies exist and are excluded


def test_selective_activation_marks_walks_in_empty_leaves():
    """With MPG_FLAG_SELECTIVE a walk is INACTIVE (w = 0, left to path tracing) exactly when
    the leaf whose box holds its (x_D, x_L) has no own sample; every other walk is unchanged."""
    w = W.config4(n_side=32, grid_n=32, guide="stree")
    r = _records(20000, seed=5)
    keep = (r["xD"][:, 0] < -3.0) | (r["xD"][:, 0] > 6.0)   # a gap without samples between two regions
    r["w"][~keep] = 0.0
    G = O.stree_build(r)
    s = O.OracleScene(w)
    s.set_stree(G)
    ids = np.arange(w.n_walks)
    on = s.walks(ids, s.opts(selective=1))
    off = s.walks(ids, s.opts(selective=0))
    inact = on["status"] == 6
    assert 50 < inact.sum() < w.n_walks - 50
    act = ~inact
    for f in ("status", "iters", "trials", "G", "T", "w", "pos"):
        assert np.array_equal(on[f][act], off[f][act]), f
    assert (on["w"][inact] == 0).all() and (on["trials"][inact] == 0).all()
    K = _key(r)
    valid = (r["w"] > 0) & (r["type"] >= 0)
    boxes = _leaf_boxes(G, K, valid)
    own = G["leaf_own"]
    key = np.concatenate([w.xD[ids // w.spp], on["xL"].astype(np.float32)], axis=1) + np.float32(0.0)
    for q in range(len(ids)):
        leaves = [l for l in range(G["n_leaves"]) if _inside(key[q], boxes[l])]
        if len(leaves) != 1:                           # outside the root box: the boundary leaf decides
            continue
        assert inact[q] == (own[leaves[0]] == 0), q
