"""Pins of the C oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it pins.  None of them compares the oracle with
itself: expected values come from closed forms (tests/closed_forms.py), NVIDIA's
own Philox, brute force, finite differences, or probability laws.
"""
import dataclasses
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12818_b200 import workloads as W
from tests import closed_forms as CF

HERE = os.path.dirname(os.path.abspath(__file__))
ETA_W = float(np.float32(1.33))   # the scene stores eta in fp32


@pytest.fixture(scope="module")
def cfg0():
    return O.OracleScene(W.config0())


# ---------------------------------------------------------------------------
# RNG: Philox4x32-10 == curand_Philox4x32_10 (library routine), 2^20 counters
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("key", [(0, 0), (0x12345678, 0x9ABCDEF0)])
def test_philox_matches_curand(tmp_path, key):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "philox_ref")
    subprocess.check_call([nvcc, "-O2", "-Wno-deprecated-gpu-targets", "-o", exe,
                           os.path.join(HERE, "golden", "philox_curand_ref.cu")])
    n = 1 << 20
    out = str(tmp_path / "ref.bin")
    subprocess.check_call([exe, str(n), str(key[0]), str(key[1]), out])
    ref = np.fromfile(out, np.uint32).reshape(n, 4)
    i = np.arange(n, dtype=np.uint64)
    ctr = np.stack([i, (i * 2654435761) & 0xFFFFFFFF, i % 40, (i * 40503) & 0xFFFFFFFF], -1).astype(np.uint32)
    got = O.philox(ctr, key)
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------------------
# Fresnel / scattering closed forms
# ---------------------------------------------------------------------------
def test_fresnel_closed_forms():
    assert O.fresnel(1.0, 1.0, 1.5) == pytest.approx(0.04, abs=1e-15)
    assert (1 - O.fresnel(1.0, 1.0, 1.5)) ** 2 == pytest.approx(0.9216, abs=1e-14)
    assert O.fresnel(np.cos(np.radians(60)), 1.5, 1.0) == 1.0                  # S:66 TIR
    crit = np.arcsin(1 / 1.5)
    assert O.fresnel(np.cos(crit - 1e-6), 1.5, 1.0) < 1.0
    # Brewster angle: r_p = 0, so F = r_s^2/2
    tb = np.arctan(1.5)
    ci, ct = np.cos(tb), np.cos(np.arcsin(np.sin(tb) / 1.5))
    rs = (ci - 1.5 * ct) / (ci + 1.5 * ct)
    assert O.fresnel(ci, 1.0, 1.5) == pytest.approx(0.5 * rs * rs, rel=1e-12)
    # transmittance is the same from both sides (Stokes relations)
    rng = np.random.default_rng(1)
    for th in rng.uniform(0, 1.5, 50):
        tt = np.arcsin(np.sin(th) / 1.5)
        assert 1 - O.fresnel(np.cos(th), 1.0, 1.5) == pytest.approx(1 - O.fresnel(np.cos(tt), 1.5, 1.0), rel=1e-12)


def test_scatter_closed_forms():
    r = O.scatter(0, 1, 1, [0, 0, -1], [0, 0, 1])
    assert np.allclose(r, [0, 0, 1])
    r = O.scatter(0, 1, 1, np.array([1, 0, -1]) / np.sqrt(2), [0, 0, 1])
    assert np.allclose(r, np.array([1, 0, 1]) / np.sqrt(2))
    assert np.allclose(O.scatter(1, 1.0, 1.5, [0, 0, -1], [0, 0, 1]), [0, 0, -1])
    d = np.array([0.3, 0.1, -0.9]) / np.linalg.norm([0.3, 0.1, -0.9])
    assert np.allclose(O.scatter(1, 1.0, 1.0, d, [0, 0, 1]), d)
    d60 = np.array([np.sin(np.radians(60)), 0, np.cos(np.radians(60))])
    assert O.scatter(1, 1.5, 1.0, d60, [0, 0, 1]) is None                       # S:66 TIR
    rng = np.random.default_rng(2)
    for _ in range(200):                                                        # S:70 tangential continuity
        n = rng.normal(size=3); n /= np.linalg.norm(n)
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        e1, e2 = rng.uniform(1, 2, 2)
        t = O.scatter(1, e1, e2, d, n)
        if t is None:
            continue
        assert np.allclose(e1 * (d - np.dot(d, n) * n), e2 * (t - np.dot(t, n) * n), atol=1e-12)
        rr = O.scatter(0, 1, 1, O.scatter(0, 1, 1, d, n), n)                     # S:57 involution
        assert np.allclose(rr, d, atol=1e-12)


# ---------------------------------------------------------------------------
# intersection and BVH == brute force
# ---------------------------------------------------------------------------
def _mirror_workload(light=None):
    quad = W.Surface(W.SURF_QUAD, W.MAT_CONDUCTOR, reflectance=1.0, origin=(-5.0, -5.0, 0.0),
                     edge_u=(10.0, 0.0, 0.0), edge_v=(0.0, 10.0, 0.0))
    sph = W.Surface(W.SURF_SPHERE, W.MAT_CONDUCTOR, center=(0.0, 0.0, 10.0), radius=1.0)
    light = light or W.Light(W.LIGHT_POINT, 1.0, position=(2.0, 0.0, 1.0))
    xD = np.array([[0.0, 0.0, 1.0]], np.float32)
    nD = np.array([[0.0, 0.0, 1.0]], np.float32)
    return W.Workload("mirror", [quad, sph], [light], xD, nD, 1, W.SeedSpec(W.SEED_CAP, 1, 1, 0), W.WalkOpts())


def test_intersection_closed_forms():
    s = O.OracleScene(_mirror_workload())
    surf, t, prim, p = s.closest([0, 0, 1], [0, 0, -1])
    assert surf == 0 and np.allclose(p, [0, 0, 0]) and t == pytest.approx(1.0)
    surf, t, prim, p = s.closest([0, 0, 10], [1, 0, 0])                       # S:47 (inside sphere)
    assert surf == 1 and np.allclose(p, [1, 0, 10])
    surf, *_ = s.closest([0, 0, 1], [1, 0, 0])                                # S:48 parallel
    assert surf == -1


@pytest.mark.parametrize("which", ["icosphere", "heightfield", "slabs"])
def test_bvh_equals_brute_force(which):
    if which == "icosphere":
        w = W.config1(n_side=4)
    elif which == "heightfield":
        w = W.config2(n_side=4, grid_n=48)
    else:
        w = W.config3(n_side=4, grid_n=24)
    s = O.OracleScene(w)
    pos, *_ = w.mesh_arrays()
    lo, hi = pos.min(0), pos.max(0)
    rng = np.random.default_rng(3)
    nhit = 0
    for _ in range(1500):
        o = rng.uniform(lo - 1, hi + 1)
        tgt = rng.uniform(lo, hi)
        d = (tgt - o) / np.linalg.norm(tgt - o)
        a = s.closest(o, d, use_bvh=True)
        b = s.closest(o, d, use_bvh=False)
        assert a[0] == b[0] and a[2] == b[2]
        if a[0] >= 0:
            nhit += 1
            assert a[1] == b[1]
    assert nhit > 500


# ---------------------------------------------------------------------------
# constraint: SPEC.md:197-199 (sign per reading R1)
# ---------------------------------------------------------------------------
def test_constraint_spec_examples():
    s = O.OracleScene(_mirror_workload())
    ok, C, J = s.constraint(1, 0, [0, 0, 1], [2, 0, 1], [[1, 0, 0]], [-1], [0])
    assert ok and np.allclose(C, 0, atol=1e-15)
    ok, C, J = s.constraint(1, 0, [0, 0, 1], [3, 0, 1], [[1, 0, 0]], [-1], [0])
    assert ok and np.max(np.abs(C)) > 1e-2
    # flat slab, normal incidence, collinear TT chain -> residual 0
    top = W.Surface(W.SURF_QUAD, W.MAT_DIELECTRIC, eta_in=1.5, eta_out=1.0, origin=(-5, 1.0, -5),
                    edge_u=(0, 0, 10), edge_v=(10, 0, 0))       # normal +y
    bot = W.Surface(W.SURF_QUAD, W.MAT_DIELECTRIC, eta_in=1.5, eta_out=1.0, origin=(-5, 0.0, -5),
                    edge_u=(10, 0, 0), edge_v=(0, 0, 10))       # normal -y
    w = dataclasses.replace(_mirror_workload(), surfaces=[bot, top])
    s2 = O.OracleScene(w)
    ok, C, J = s2.constraint(2, 3, [0.3, -2, 0.2], [0.3, 5, 0.2], [[0.3, 0, 0.2], [0.3, 1, 0.2]], [-1, -1], [0, 1])
    assert ok and np.allclose(C, 0, atol=1e-14)


def _converged_chains(s, w, n_walks, stride=1):
    r = s.walks(np.arange(0, n_walks * stride, stride))
    idx = np.nonzero(r["status"] == 0)[0]
    return r, idx


@pytest.mark.parametrize("which", ["cfg0", "cfg1a", "cfg1", "cfg2", "cfg3"])
def test_jacobian_matches_fd_at_admissible_chains(which):
    """Analytic blocks == central FD of C at admissible chains (reading R3; SPEC.md:290
    restricted to admissible chains, where the frame-twist term vanishes)."""
    w = {"cfg0": lambda: W.config0(16, 4), "cfg1a": lambda: W.config1(16, 1, analytic=True),
         "cfg1": lambda: W.config1(24, 1), "cfg2": lambda: W.config2(16, 4, grid_n=96),
         "cfg3": lambda: W.config3(32, 1, grid_n=48)}[which]()
    s = O.OracleScene(w)
    r, idx = _converged_chains(s, w, w.n_walks)
    assert len(idx) >= 5
    k, tau = w.seed.k, w.seed.tau
    worst = 0.0
    for q in idx[:12]:
        xD = w.xD[r["walk"][q] // w.spp].astype(np.float64)
        xL = r["xL"][q]
        pos, prim, surf = r["pos"][q], r["prim"][q], r["surf"][q]
        ok, C0, J = s.constraint(k, tau, xD, xL, pos, prim, surf)
        assert ok
        h = 1e-6
        for j in range(k):
            sg, tg = s.tangent_basis(prim[j], surf[j], pos[j])
            for c, v in enumerate((sg, tg)):
                pp, pm = pos.copy(), pos.copy()
                pp[j] += h * v
                pm[j] -= h * v
                _, Cp, _ = s.constraint(k, tau, xD, xL, pp, prim, surf)
                _, Cm, _ = s.constraint(k, tau, xD, xL, pm, prim, surf)
                fd = (Cp - Cm) / (2 * h)
                an = J[:, 2 * j + c]
                scale = max(1.0, np.max(np.abs(J)))
                worst = max(worst, np.max(np.abs(fd - an)) / scale)
    assert worst < 1e-5, worst


# ---------------------------------------------------------------------------
# Newton: idempotence, plane mirror, quadratic convergence
# ---------------------------------------------------------------------------
def test_idempotence(cfg0):
    r, idx = _converged_chains(cfg0, cfg0.w, 2000)
    for q in idx[:50]:
        xD = cfg0.w.xD[r["walk"][q] // cfg0.w.spp]
        st, it, pos, prim, surf, _ = cfg0.newton_chain(1, 0, xD, r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q])
        assert st == 0 and it == 0 and np.allclose(pos, r["pos"][q], atol=0)


def test_plane_mirror_converges_to_image_point():
    s = O.OracleScene(_mirror_workload())
    rng = np.random.default_rng(4)
    tight = s.opts(tol=1e-9, max_iters=60)
    for _ in range(50):
        tgt = np.array([rng.uniform(-2, 3), rng.uniform(-2, 2), 0.0])
        out = s.walk_from_target([0, 0, 1], [0, 0, 1], [2, 0, 1], tgt, opts=tight)
        assert out["status"] == 0
        assert np.allclose(out["pos"][0], [1, 0, 0], atol=1e-6)
    # seeds near the solution: <= 2 iterations
    for _ in range(20):
        tgt = np.array([1 + rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05), 0.0])
        out = s.walk_from_target([0, 0, 1], [0, 0, 1], [2, 0, 1], tgt)
        assert out["status"] == 0 and out["iters"] <= 2


def test_quadratic_convergence_sphere(cfg0):
    """Local quadratic convergence (PAPER.md:362 footnote): residual
    after one Newton step ~ d^2, log-log slope in [1.8, 2.2]."""
    w = cfg0.w
    r, idx = _converged_chains(cfg0, w, 3000)
    q = idx[0]
    xD = w.xD[r["walk"][q] // w.spp].astype(np.float64)
    xL = r["xL"][q]
    p0 = r["pos"][q][0]
    v = np.cross(p0, [0.3, 0.5, 0.7]); v /= np.linalg.norm(v)
    ds = np.logspace(-4.5, -2.5, 9)
    res = []
    for d in ds:
        p = p0 + d * v
        p = p / np.linalg.norm(p)
        opts = cfg0.opts(max_iters=1, tol=0.0)
        st, it, pos, prim, surf, hist = cfg0.newton_chain(1, 0, xD, xL, [p], [-1], [0], opts)
        res.append(hist[1])
    slope = np.polyfit(np.log(ds), np.log(res), 1)[0]
    assert 1.8 <= slope <= 2.2, slope


# ---------------------------------------------------------------------------
# converged chains == closed-form solutions (Alhazen, in-plane TT, Snell plane)
# ---------------------------------------------------------------------------
def test_cfg0_chains_are_alhazen_points(cfg0):
    w = cfg0.w
    recv = np.arange(0, w.n_recv, 7)
    ids = (recv[:, None] * w.spp + np.arange(w.spp)[None, :]).ravel()
    r = cfg0.walks(ids, cfg0.opts(tol=1e-11, max_iters=40))   # tight tol: pins the zero set itself
    ext = cfg0.extent
    nconv = 0
    for ri in recv:
        sel = np.nonzero(r["walk"] // w.spp == ri)[0]
        xL = r["xL"][sel[0]]
        pts = CF.alhazen_points([0, 0, 0], 1.0, w.xD[ri], xL)
        conv = sel[r["status"][sel] == 0]
        if len(pts) == 0:
            assert len(conv) == 0
            continue
        assert len(pts) == 1
        for q in conv:
            nconv += 1
            assert np.linalg.norm(r["pos"][q][0] - pts[0]) < 1e-6 * ext
    assert nconv > 500


def test_twin1a_chains_are_inplane_TT_roots():
    w = W.config1(32, 4, analytic=True)
    w.opts.tol, w.opts.max_iters = 1e-11, 40
    s = O.OracleScene(w)
    r, idx = _converged_chains(s, w, w.n_walks)
    assert len(idx) > 50
    for q in idx[:60]:
        xD = w.xD[r["walk"][q] // w.spp]
        sols = CF.tt_sphere_chains([0, 0, 0], 1.0, 1.5, xD, r["xL"][q], near=r["pos"][q][0])
        assert sols
        d = min(np.linalg.norm(r["pos"][q][0] - a) + np.linalg.norm(r["pos"][q][1] - b) for a, b in sols)
        assert d < 1e-8 * s.extent


def test_twin2a_snell_point_and_G():
    w = W.config2(16, 4, flat=True, grid_n=64)
    w.opts.tol, w.opts.max_iters = 1e-11, 40
    s = O.OracleScene(w)
    r, idx = _converged_chains(s, w, w.n_walks)
    assert len(idx) > 50
    for q in idx:
        xD = w.xD[r["walk"][q] // w.spp]
        x1, G = CF.snell_plane(xD, r["xL"][q], ETA_W, 1.0)
        assert np.linalg.norm(r["pos"][q][0] - x1) < 1e-10 * s.extent
        assert r["G"][q] == pytest.approx(G, rel=1e-9)


def test_snell_layers_closed_form_special_cases():
    """The layered closed form reduces to the textbook cases: one interface is
    tests/closed_forms.snell_plane's Snell point; index-matched layers give a
    straight segment with G = cos^3 t / H^2 (= cos/r^2) and kappa = 1; normal
    incidence gives kappa = (1 - 0.04)^2 per slab."""
    xD, xL = np.array([0.2, -1.0, -0.3]), np.array([0.9, 2.5, 0.4])
    pts = CF.snell_layers(xD, xL, [0.0], [1.33, 1.0])
    x1, _ = CF.snell_plane(xD, xL, 1.33, 1.0)
    assert np.allclose(pts[0], x1, atol=1e-12)
    pts, G, kappa = CF.snell_layers(xD, xL, [0.0, 0.1, 0.7], [1.0] * 4, with_G=True)
    d = xL - xD
    for p in pts:                                             # on the segment x_D x_L
        assert np.linalg.norm(np.cross(p - xD, d)) < 1e-12
    r = np.linalg.norm(d)
    assert G == pytest.approx((d[1] / r) / r ** 2, rel=1e-12) and kappa == pytest.approx(1.0, abs=1e-15)
    _, _, kappa = CF.snell_layers(xD, xD + [1e-9, 3.5, 0.0], [0.0, 0.1, 0.35, 0.45], [1.0, 1.5, 1.0, 1.5, 1.0],
                                  with_G=True)
    assert kappa == pytest.approx(0.9216 ** 2, rel=1e-9)


def test_twin3a_k6_chains_are_layered_snell_points():
    """k = 6 TTTTTT through three planar glass slabs (twin of configs[3]): every
    converged chain is the unique straight-up refraction path fixed by Snell's
    invariant eta sin t (closed form tests/closed_forms.snell_layers).  Pins the
    6-block tridiagonal elimination and back-substitution, the
    sequential reprojection through six interfaces (reading R5), the analytic GGT
    (Eq. 2) and kappa = product of six Fresnel transmittances."""
    w = W.config3(24, 1, grid_n=16, flat=True)
    w.opts.tol, w.opts.max_iters = 1e-11, 60
    s = O.OracleScene(w)
    ys = [float(srf.positions[0, 1]) for srf in w.surfaces]   # fp32 planes, bottom to top
    assert ys == sorted(ys) and len(ys) == 6
    etas = [1.0, 1.5, 1.0, 1.5, 1.0, 1.5, 1.0]
    r, idx = _converged_chains(s, w, w.n_walks)
    assert len(idx) > 50
    for q in idx:
        xD = w.xD[r["walk"][q] // w.spp]
        ref, G, kappa = CF.snell_layers(xD, r["xL"][q], ys, etas, with_G=True)
        assert np.abs(np.asarray(r["pos"][q][:6]) - ref).max() < 1e-9 * s.extent
        assert r["G"][q] == pytest.approx(G, rel=1e-9)                # Eq. 2 GGT, k = 6
        assert r["T"][q] == pytest.approx(kappa * G, rel=1e-9)        # T = kappa G I, I = 1


# ---------------------------------------------------------------------------
# GGT (Eq. 2): unfold, Coddington, FD re-convergence, reciprocity
# ---------------------------------------------------------------------------
def test_ggt_plane_mirror_unfold():
    eu = np.array([0.625, 0.0, 0.0])   # fp32-exact so both sides see the same plane
    ev = np.array([0.0, 0.375, -0.5])
    light = W.Light(W.LIGHT_QUAD, 1.0, position=(2.0, 0.5, 1.5), edge_u=tuple(eu), edge_v=tuple(ev))
    s = O.OracleScene(_mirror_workload(light))
    xD, nD, xL = np.array([0.0, 0.0, 1.0]), np.array([0.0, 0.0, 1.0]), np.array([2.0, 0.5, 1.5])
    out = s.walk_from_target(xD, nD, xL, [0.8, 0.1, 0.0], opts=s.opts(tol=1e-12, max_iters=40))
    assert out["status"] == 0
    img = np.array([0.0, 0.0, -1.0])
    d = np.linalg.norm(xL - img)
    u = (xL - img) / d
    nL = np.cross(eu, ev); nL /= np.linalg.norm(nL)
    wD = (out["pos"][0] - xD) / np.linalg.norm(out["pos"][0] - xD)
    Gc = abs(np.dot(nD, wD)) * abs(np.dot(nL, u)) / d ** 2
    G = s.ggt(1, 0, xD, nD, xL, out["pos"], out["prim"], out["surf"])
    assert G == pytest.approx(Gc, rel=1e-10)


def test_ggt_sphere_coddington(cfg0):
    w = cfg0.w
    r = cfg0.walks(np.arange(6000), cfg0.opts(tol=1e-11, max_iters=40))
    idx = np.nonzero(r["status"] == 0)[0]
    for q in idx[:100]:
        xD = w.xD[r["walk"][q] // w.spp]
        Gc = CF.coddington_G([0, 0, 0], 1.0, xD, [0, 1, 0], r["xL"][q], r["pos"][q][0])
        assert r["G"][q] == pytest.approx(Gc, rel=1e-9)
        assert r["T"][q] == pytest.approx(Gc, rel=1e-9)      # kappa = rho = 1, I = 1


@pytest.mark.parametrize("which", ["cfg1", "cfg2", "cfg3"])
def test_ggt_analytic_equals_fd_reconvergence(which):
    """FD re-convergence GGT, invariant to halving delta, equals
    the analytic manifold-tangent GGT (reading R11)."""
    w = {"cfg1": lambda: W.config1(24, 1), "cfg2": lambda: W.config2(16, 4, grid_n=96),
         "cfg3": lambda: W.config3(32, 1, grid_n=48)}[which]()
    w.opts.tol, w.opts.max_iters = 1e-12, 60     # G is evaluated at the exact chain
    s = O.OracleScene(w)
    r, idx = _converged_chains(s, w, w.n_walks)
    k, tau = w.seed.k, w.seed.tau
    checked = 0
    for q in idx[:15]:
        xD = w.xD[r["walk"][q] // w.spp]
        a = s.ggt(k, tau, xD, w.nD[0], r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q], method=0)
        f1 = s.ggt(k, tau, xD, w.nD[0], r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q], method=1, delta=2e-6)
        f2 = s.ggt(k, tau, xD, w.nD[0], r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q], method=1, delta=1e-6)
        if f1 < 0 or f2 < 0:
            continue        # re-convergence crossed a triangle edge / failed
        checked += 1
        assert f1 == pytest.approx(f2, rel=1e-5)
        assert a == pytest.approx(f2, rel=1e-5)
        assert a == pytest.approx(r["G"][q], rel=1e-12)
    assert checked >= 5


@pytest.mark.parametrize("which", ["water_flat", "sphere_TT"])
def test_ggt_reciprocity(which):
    """eta_D^2 G(D<-L) = eta_L^2 G(L<-D) (etendue conservation; SURVEY 8(c) pin).
    Exact for integrable normal fields (flat water, analytic sphere); Phong
    shading normals are not integrable and break it at O(curvature error)."""
    if which == "water_flat":
        w = W.config2(8, 1, flat=True, grid_n=32)
        etaD, etaL = ETA_W, 1.0
    else:
        w = W.config1(16, 2, analytic=True)
        etaD, etaL = 1.0, 1.0
    w.opts.tol, w.opts.max_iters = 1e-12, 60
    s = O.OracleScene(w)
    r, idx = _converged_chains(s, w, w.n_walks)
    assert len(idx) >= 3
    k, tau = w.seed.k, w.seed.tau
    for q in idx[:5]:
        xD = w.xD[r["walk"][q] // w.spp].astype(np.float64)
        xL = r["xL"][q]
        Gf = r["G"][q]
        # reversed: receiver at x_L (normal -y), area light through x_D facing +y
        rev = dataclasses.replace(w, lights=[W.Light(W.LIGHT_QUAD, 1.0, position=tuple(xD), edge_u=(1.0, 0.0, 0.0),
                                                     edge_v=(0.0, 0.0, -1.0))])
        s2 = O.OracleScene(rev)
        Gr = s2.ggt(k, tau, xL, [0, -1, 0], xD, r["pos"][q][::-1], r["prim"][q][::-1], r["surf"][q][::-1])
        assert etaD ** 2 * Gf == pytest.approx(etaL ** 2 * Gr, rel=1e-8)


def test_kappa_closed_forms():
    w = W.config1(4, 1, analytic=True)
    s = O.OracleScene(w)
    kap = s.kappa(2, 3, [0, -1.2, 0], [0, 5, 0], [[0, -1, 0], [0, 1, 0]], [-1, -1], [0, 0])
    assert kap == pytest.approx(0.9216, rel=1e-12)
    w2 = W.config2(4, 1, flat=True, grid_n=16)
    s2 = O.OracleScene(w2)
    pos, nrm, idx, ts, _ = w2.mesh_arrays()
    surf, t, prim, p = s2.closest([3.3, -2, 4.1], [0, 1, 0])
    kap = s2.kappa(1, 1, [3.3, -2, 4.1], [3.3, 8, 4.1], [p], [prim], [surf])
    F = ((ETA_W - 1) / (ETA_W + 1)) ** 2
    assert kap == pytest.approx((1 - F) * ETA_W ** 2, rel=1e-12)                  # radiance eta^2 law (R12)


# ---------------------------------------------------------------------------
# trials and estimator (Eqs. 3, 15): E[k] = 1/P_basin, E[w] = sum T
# ---------------------------------------------------------------------------
def _single_receiver(w, ri, spp):
    return dataclasses.replace(w, xD=w.xD[ri:ri + 1].copy(), nD=w.nD[ri:ri + 1].copy(), spp=spp)


def _cap_grid_targets(xD, n):
    xD = np.asarray(xD, np.float64)
    L = np.linalg.norm(xD)
    a = xD / L
    cmin = 1.0 / L
    b1 = np.cross(a, [0.3, 0.7, 0.1]); b1 /= np.linalg.norm(b1)
    b2 = np.cross(a, b1)
    u = (np.arange(n) + 0.5) / n
    U1, U2 = np.meshgrid(u, u, indexing="ij")
    ct = 1 - U1 * (1 - cmin)
    st = np.sqrt(1 - ct * ct)
    ph = 2 * np.pi * U2
    d = ct[..., None] * a + st[..., None] * (np.cos(ph)[..., None] * b1 + np.sin(ph)[..., None] * b2)
    return d.reshape(-1, 3)


def test_trial_count_is_reciprocal_basin_fraction(cfg0):
    w = cfg0.w
    ri = 64 * 30 + 10
    xD = w.xD[ri]
    tg = _cap_grid_targets(xD, 96)
    conv = [cfg0.walk_from_target(xD, [0, 1, 0], [0, 4, 0], t)["status"] == 0 for t in tg]
    P = np.mean(conv)
    assert 0.1 < P < 0.9
    ws = O.OracleScene(_single_receiver(w, ri, 4000))
    r = ws.walks(np.arange(4000))
    c = r["status"] == 0
    n = c.sum()
    assert abs(c.mean() - P) < 4 * np.sqrt(P * (1 - P) / 4000) + 1.0 / 96
    kmean = r["trials"][c].mean()
    se = np.sqrt((1 - P) / P ** 2 / n)
    assert abs(kmean - 1 / P) < 4 * se + 0.05 / P


def test_estimator_unbiased_cfg0(cfg0):
    """Eq. 3/4: mean w over seeds = sum over admissible chains of T (here one
    Alhazen chain with Coddington G, or none)."""
    w = cfg0.w
    for ri in (64 * 30 + 10, 64 * 50 + 33, 64 * 12 + 40, 64 * 63 + 0):
        ws = O.OracleScene(_single_receiver(w, ri, 3000))
        r = ws.walks(np.arange(3000))
        pts = CF.alhazen_points([0, 0, 0], 1.0, w.xD[ri], [0, 4, 0])
        if not pts:
            assert np.all(r["w"] == 0)
            continue
        T = CF.coddington_G([0, 0, 0], 1.0, w.xD[ri], [0, 1, 0], [0, 4, 0], pts[0])
        m, se = r["w"].mean(), r["w"].std() / np.sqrt(len(r["w"]))
        assert abs(m - T) < 3.5 * se, (m, T, se)


def test_estimator_unbiased_twin3a_k6():
    """Eq. 3 with the reciprocal-probability weight (Eq. 15) on
    k = 6 guided seeds: mean w over seeds = T = kappa G I of the one layered-Snell
    chain (closed form), whatever the guide's seed density."""
    w = W.config3(8, 1, grid_n=16, flat=True)
    ys = [float(srf.positions[0, 1]) for srf in w.surfaces]
    etas = [1.0, 1.5, 1.0, 1.5, 1.0, 1.5, 1.0]
    for ri in (8 * 3 + 3, 8 * 4 + 2, 8 * 2 + 5):
        ws = O.OracleScene(_single_receiver(w, ri, 2000))
        r = ws.walks(np.arange(2000))
        assert r["truncated"].sum() == 0
        pts, G, kappa = CF.snell_layers(w.xD[ri], r["xL"][0], ys, etas, with_G=True)
        assert np.all(np.abs(pts[:, [0, 2]]) < 0.95)        # chain inside the meshes
        m, se = r["w"].mean(), r["w"].std() / np.sqrt(len(r["w"]))
        assert se < 0.2 * kappa * G
        assert abs(m - kappa * G) < 3.5 * se, (m, kappa * G, se)


def test_cfg4_mirror_sphere_chains_closed_form():
    """configs[4] (mixed scene, three lights, chain length and type drawn per walk):
    every converged k = 1 chain on the mirror sphere lies at the Alhazen point for
    its light sample, with G = Coddington (point light) or Coddington x cos t_L
    (quad lights), and T = G (rho = 1, L_e = I = 1, unit-area lights; Eq. 2)."""
    w = W.config4(n_side=160, grid_n=32)
    w.opts.tol, w.opts.max_iters, w.opts.max_iters_long = 1e-11, 40, 60
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks))
    sel = np.nonzero((r["status"] == 0) & (r["k"] == 1) & (r["surf"][:, 0] == 0))[0]
    n_point = 0
    for q in sel:
        xD, xL = w.xD[r["walk"][q] // w.spp], r["xL"][q]
        pts = CF.alhazen_points([-5, 0, 2.5], 1.0, xD, xL)
        p = r["pos"][q][0]
        assert min(np.linalg.norm(p - a) for a in pts) < 1e-10 * s.extent
        point = np.allclose(xL, [-5.0, 4.0, 2.5])
        n_point += point
        G = CF.mirror_sphere_G([-5, 0, 2.5], 1.0, xD, [0, 1, 0], xL, p, None if point else [0, 1, 0])
        assert r["G"][q] == pytest.approx(G, rel=1e-8)
        assert r["T"][q] == pytest.approx(G, rel=1e-8)
    assert len(sel) > 30 and 5 < n_point < len(sel)


def test_dense_grid_enumeration_is_complete(cfg0):
    """dense seed grid, dedupe by same_chain, count stable under
    resolution doubling; equals the Alhazen root count."""
    w = cfg0.w
    for ri in (64 * 30 + 10, 64 * 5 + 60, 64 * 63 + 63):
        xD = w.xD[ri]
        counts = []
        for n in (48, 96):
            chains = []
            for t in _cap_grid_targets(xD, n):
                o = cfg0.walk_from_target(xD, [0, 1, 0], [0, 4, 0], t)
                if o["status"] == 0 and not any(np.linalg.norm(o["pos"][0] - c) < 1e-4 * cfg0.extent for c in chains):
                    chains.append(o["pos"][0])
            counts.append(len(chains))
        assert counts[0] == counts[1] == len(CF.alhazen_points([0, 0, 0], 1.0, xD, [0, 4, 0]))


# ---------------------------------------------------------------------------
# seeds and guide tables (Eqs. 8, 13)
# ---------------------------------------------------------------------------
def test_guide_tables_are_defensive_mixture():
    rng = np.random.default_rng(5)
    E = np.concatenate([rng.lognormal(0, 1, (4, 1024)), np.zeros((1, 1024))]).astype(np.float32)
    Ed = rng.dirichlet(np.full(4096, 0.3), 3).astype(np.float32)
    for EE in (E, Ed):
        pf = O.guide_tables(EE).astype(np.float64)
        N = EE.shape[1]
        for c in range(EE.shape[0]):
            p = np.diff(np.concatenate([[0.0], pf[c]])) / pf[c, -1]
            assert p.sum() == pytest.approx(1.0, abs=1e-12)
            if EE[c].sum() == 0:
                assert np.allclose(p, 1.0 / N)                     # learned branch absent
                continue
            assert np.all(p >= 0.5 / N * (1 - 1e-12))              # defensive bound
            q = EE[c].astype(np.float64) / EE[c].sum()
            learned = 2 * p - 1.0 / N                               # Eq. 13 with alpha = 1/2
            sumW = 2 ** 20                                          # lower bound on sum of W
            assert np.all(np.abs(learned - q) <= (1.0 + q * N) / sumW + 1e-12)


def test_guided_seed_bins_follow_table():
    """Integer-CDF bin draws follow the defensive table W'/sum W' (chi^2, 1023 dof)."""
    n = 60000
    w = _single_receiver(W.config2(4, 1, grid_n=16), 5, n)
    s = O.OracleScene(w)
    xD = w.xD[0]
    cx = int(np.floor(xD[0] * 16 / 10.0))
    cz = int(np.floor(xD[2] * 16 / 10.0))
    bins = np.array([s.seed(i)[4] for i in range(n)])
    pf = s.prefix[cz * 16 + cx].astype(np.float64)
    p = np.diff(np.concatenate([[0.0], pf])) / pf[-1]
    cnt = np.bincount(bins, minlength=1024)
    exp = p * n
    chi2 = ((cnt - exp) ** 2 / exp).sum()
    assert chi2 < 1023 + 6 * 45          # mean 1023, sd ~45
    # targets lie in the drawn bin of the (u,v) map on the plane y = uv_plane_y
    for i in range(200):
        ok, xL, pdf, tgt, b = s.seed(i)
        u, v = tgt[0] / 10.0, tgt[2] / 10.0
        assert int(u * 32) == b % 32 and int(v * 32) == b // 32 and tgt[1] == 0.0


def test_cap_seeds_uniform_on_visible_cap():
    w = W.config0(1, 20000)
    w = dataclasses.replace(w, xD=np.array([[1.7, -1.5, -0.4]], np.float32), nD=w.nD[:1])
    s = O.OracleScene(w)
    tg = np.array([s.seed(i)[3] for i in range(20000)], np.float64)
    xD = w.xD[0].astype(np.float64)
    a = xD / np.linalg.norm(xD)
    cmin = 1 / np.linalg.norm(xD)
    ct = tg @ a / np.linalg.norm(tg, axis=1)
    assert np.all(ct > cmin - 1e-6)
    u = np.sort((1 - ct) / (1 - cmin))
    ks = np.max(np.abs(u - (np.arange(len(u)) + 0.5) / len(u)))
    assert ks < 1.63 / np.sqrt(len(u)) + 1e-3                                   # KS at ~1%


def test_triangle_seeds_front_facing_and_uniform():
    w = W.config1(1, 30000)
    s = O.OracleScene(w)
    pos, nrm, idx, *_ = w.mesh_arrays()
    xD = w.xD[0].astype(np.float64)
    tris, bary = [], []
    nfail = 0
    for i in range(30000):
        ok, xL, pdf, tgt, b = s.seed(i)
        if not ok:
            nfail += 1
            continue
        v0, v1, v2 = pos[idx[b]].astype(np.float64)
        ng = np.cross(v1 - v0, v2 - v0)
        assert np.dot(xD - v0, ng) > 0
        M = np.stack([v1 - v0, v2 - v0], 1)
        lam, *_ = np.linalg.lstsq(M, tgt.astype(np.float64) - v0, rcond=None)
        bary.append(lam)
        tris.append(b)
    front = [t for t in range(idx.shape[0]) if np.dot(xD - pos[idx[t, 0]], np.cross(pos[idx[t, 1]] - pos[idx[t, 0]],
                                                                                    pos[idx[t, 2]] - pos[idx[t, 0]])) > 0]
    f = len(front) / idx.shape[0]
    pfail = (1 - f) ** 32                                                     # <= 32 rejection draws
    assert abs(nfail - 30000 * pfail) < 5 * np.sqrt(30000 * pfail) + 1
    cnt = np.bincount(tris, minlength=idx.shape[0])[front]
    exp = (30000 - nfail) / len(front)
    chi2 = ((cnt - exp) ** 2 / exp).sum()
    dof = len(front) - 1
    assert chi2 < dof + 6 * np.sqrt(2 * dof)
    bary = np.array(bary)
    assert np.allclose(bary.mean(0), [1 / 3, 1 / 3], atol=0.01)               # uniform in the triangle
    assert np.all(bary >= -1e-5) and np.all(bary.sum(1) <= 1 + 1e-5)


def test_light_samples_uniform_on_quad():
    w = W.config1(1, 20000)
    s = O.OracleScene(w)
    xs = np.array([s.seed(i)[1] for i in range(20000)])
    assert np.all(np.abs(xs[:, 0]) <= 0.5) and np.all(np.abs(xs[:, 2]) <= 0.5) and np.all(xs[:, 1] == 5.0)
    assert abs(xs[:, 0].mean()) < 0.01 and abs(xs[:, 2].mean()) < 0.01
    assert xs[:, 0].var() == pytest.approx(1 / 12, rel=0.05)
    assert s.seed(0)[2] == pytest.approx(1.0)


# ---------------------------------------------------------------------------
# configs[4]: typed direction guide and the Eq. 8 / Eq. 13 sampler (R22)
# ---------------------------------------------------------------------------
def _random_typed_hist(rng, cells=4, nb=1024):
    H = np.zeros((cells, 126, nb), np.float32)
    for c in range(1, cells):                       # cell 0 empty: learned branch absent
        for t in rng.choice(126, size=12, replace=False):
            if c == 2 and t >= 62:                  # cell 2: no mass for n = 6
                continue
            m = rng.random(nb) < 0.1
            H[c, t, m] = rng.lognormal(0, 1, m.sum()).astype(np.float32)
    return H


def test_dir_tables_are_defensive_mixtures():
    rng = np.random.default_rng(11)
    H = _random_typed_hist(rng)
    npf, tpf, dpf = O.guide_dir_tables(H)
    P0 = np.array([1, 1, 1, 1, 1, 0.95]) / 5.95               # RR from bounce 5, gamma 0.95
    for c in range(H.shape[0]):
        Pn = np.diff(np.concatenate([[0.0], npf[c].astype(np.float64)])) / float(npf[c, -1])
        E = H[c].astype(np.float64).sum(1)
        En = np.array([E[(1 << n) - 2:(1 << (n + 1)) - 2].sum() for n in range(1, 7)])
        if En.sum() == 0:
            assert np.allclose(Pn, P0, atol=1e-15)               # learned branch absent
            continue
        Pe = 2 * Pn - P0                                        # Eq. 13, alpha = 1/2
        assert np.all(Pn >= 0.5 * P0 * (1 - 1e-12))               # defensive bound
        assert np.allclose(Pe, En / En.sum(), atol=1e-5)         # Eq. 10 within 2^-20 quantisation
        for n in range(1, 7):
            g0, gn = (1 << n) - 2, 1 << n
            Eg = E[g0:g0 + gn]
            w = np.diff(np.concatenate([[0], tpf[c, g0:g0 + gn].astype(np.float64)]))
            if Eg.sum() == 0:
                assert w.sum() == 0
            else:
                assert np.allclose(w / w.sum(), Eg / Eg.sum(), atol=1e-5)   # Eq. 11
        for t in range(126):
            d = np.diff(np.concatenate([[0], dpf[c, t].astype(np.float64)]))
            if H[c, t].sum() > 0:
                assert np.allclose(d / d.sum(), H[c, t] / H[c, t].astype(np.float64).sum(), atol=1e-5)
                assert np.all((d > 0) == (H[c, t] > 0))
            else:
                assert d.sum() == 0


def test_dir_sampler_follows_eq8_and_eq13():
    """n ~ P(n) table; the learned branch is taken with probability 1/2 when available
    (one-sample MIS, Eq. 13); learned types ~ P_e(tau|n) (Eq. 11); initializer
    directions uniform on the hemisphere (cos(theta), phi uniform; "direction")."""
    w = W.config4(n_side=4, grid_n=16)
    rng = np.random.default_rng(12)
    H = np.zeros((256, 126, 1024), np.float32)
    Hs = _random_typed_hist(rng, cells=4)
    rcv = 5
    cx = int(np.floor(((w.xD[rcv, 0] + 7.5) * 16) / 17.5)); cz = int(np.floor((w.xD[rcv, 2] * 16) / 10.0))
    H[cz * 16 + cx] = Hs[1]
    one = dataclasses.replace(w, xD=w.xD[rcv:rcv + 1].copy(), nD=w.nD[:1].copy(), spp=20000)
    s = O.OracleScene(one)
    s.set_dir_hist(H)
    npf, tpf, dpf = s.dir_tables
    c = cz * 16 + cx
    Pn = np.diff(np.concatenate([[0.0], npf[c].astype(np.float64)])) / float(npf[c, -1])
    draws = [s.seed_ex(i) for i in range(20000)]
    ns = np.array([d["n"] for d in draws])
    cnt = np.bincount(ns, minlength=7)[1:]
    chi2 = ((cnt - 20000 * Pn) ** 2 / (20000 * Pn)).sum()
    assert chi2 < 5 + 6 * np.sqrt(10)
    assert all(abs(d["Pn"] - Pn[d["n"] - 1]) < 1e-12 for d in draws[:200])
    E = Hs[1].astype(np.float64).sum(1)
    avail = [d for d in draws if E[(1 << d["n"]) - 2:(1 << (d["n"] + 1)) - 2].sum() > 0]
    frac = np.mean([d["learned"] for d in avail])
    assert abs(frac - 0.5) < 4 * np.sqrt(0.25 / len(avail))
    init = [d for d in draws if not d["learned"]]
    dirs = np.array([d["target"] for d in init], np.float64) - one.xD[0]
    u = np.sort(dirs[:, 1])
    ks = np.max(np.abs(u - (np.arange(len(u)) + 0.5) / len(u)))
    assert ks < 1.63 / np.sqrt(len(u)) + 1e-3
    phi = np.sort((np.arctan2(dirs[:, 2], dirs[:, 0]) + np.pi) / (2 * np.pi))
    assert np.max(np.abs(phi - (np.arange(len(phi)) + 0.5) / len(phi))) < 1.63 / np.sqrt(len(phi)) + 1e-3
    # learned types within the most frequent learned length follow P_e(tau|n)
    lrn = [d for d in draws if d["learned"]]
    nbest = np.bincount([d["n"] for d in lrn]).argmax()
    g0, gn = (1 << nbest) - 2, 1 << nbest
    ts = np.bincount([d["tau"] for d in lrn if d["n"] == nbest], minlength=gn)
    pt = E[g0:g0 + gn] / E[g0:g0 + gn].sum()
    m = pt > 0
    assert np.all(ts[~m] == 0)
    chi2 = ((ts[m] - ts.sum() * pt[m]) ** 2 / (ts.sum() * pt[m])).sum()
    assert chi2 < m.sum() + 6 * np.sqrt(2 * m.sum())


def run_oracle_progressive(w, iterations):
    s = O.OracleScene(w)
    out = []
    for it in range(iterations):
        r = s.walks(np.arange(w.n_walks), s.opts(walk_id_base=it * w.n_walks))
        out.append(r)
        H = s.accumulate_dir(r["status"], r["w"], r["pos"][:, 0].astype(np.float32), r["k"], r["tau"])
        s.set_dir_hist(H.astype(np.float32))            # last iteration only (P:426 footnote)
    return out


def test_progressive_loop_learns():
    """The guided distribution approaches the energy distribution (Eq. 5): after
    the initializer-only iteration 0, guided iterations convert far more seeds into
    admissible chains and need fewer reciprocal trials."""
    w = W.config4(n_side=48, grid_n=64)
    res = run_oracle_progressive(w, 3)
    conv = [np.mean(r["status"] == 0) for r in res]
    tri = [r["trials"][r["trials"] > 0].mean() for r in res]
    assert conv[2] > 2 * conv[0], conv
    assert tri[2] < tri[0], tri


# ---------------------------------------------------------------------------
# R x M: M reciprocal-probability estimates averaged [R32]
# ---------------------------------------------------------------------------
def test_repeated_reciprocal_estimates_unbiased_and_lower_variance():
    """Averaging M independent geometric counts keeps E[w] (Eq. 15 stays unbiased) and cuts
    the variance of w; the solved chains (trial 0) are unchanged and every count is >= M."""
    w = dataclasses.replace(W.config0(n_side=8, spp=64))
    s = O.OracleScene(w)
    ids = np.arange(w.n_walks)
    a = s.walks(ids, s.opts())
    b = s.walks(ids, s.opts(recip_repeats=4))
    assert np.array_equal(a["status"], b["status"]) and np.array_equal(a["pos"], b["pos"])
    conv = (a["status"] == 0) & (a["T"] > 0)
    assert (b["trials"][conv] >= 4).all() and (a["trials"][conv] >= 1).all()
    # per receiver: same mean within the standard errors, lower variance
    wa = a["w"].reshape(-1, w.spp)
    wb = b["w"].reshape(-1, w.spp)
    se = np.sqrt(wa.var(1, ddof=1) / w.spp + wb.var(1, ddof=1) / w.spp)
    ok = se > 0
    z = np.abs(wa.mean(1) - wb.mean(1))[ok] / se[ok]
    assert (z < 3).mean() >= 0.95 and z.max() < 5
    assert abs(wa.mean() - wb.mean()) < 3 * np.sqrt(wa.var() / wa.size + wb.var() / wb.size)
    assert wb.var(1).mean() < 0.8 * wa.var(1).mean()


# ---------------------------------------------------------------------------
# visibility V (Eq. 2, "including the visibility function"; O8):
# closed-form occluders and brute-force any-hit
# ---------------------------------------------------------------------------
def _occlusion_closed_form(xD, p, xL, margin):
    """Twin 0v: the Alhazen chain x_D -> p -> x_L is occluded iff one of its two
    segments crosses one of the rectangles OCCLUDERS_0V (None: too close to call)."""
    hits = [CF.segment_hits_rect(a, b, R, margin) for R in W.OCCLUDERS_0V for a, b in ((xD, p), (p, xL))]
    if any(h is None for h in hits):
        return None
    return any(hits)


def test_visibility_closed_form_occluders():
    """Twin 0v (configs[0] plus two opaque diffuse rectangles): every converged walk
    is OCCLUDED with G = T = 0 exactly when a segment of its (unique) Alhazen chain
    crosses a rectangle, else CONVERGED with the Coddington G; the rectangles do not
    take part in deduction or reprojection (specular surfaces only, Eq. 6)."""
    w = W.config0(n_side=48, spp=4, occluders=True)
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks), s.opts(tol=1e-11, max_iters=40))   # tight tol: G to 1e-6
    ext = s.extent
    n = {True: 0, False: 0}
    for q in np.nonzero(np.isin(r["status"], (0, 5)))[0]:
        xD, xL = w.xD[q // w.spp].astype(np.float64), r["xL"][q]
        pts = CF.alhazen_points([0, 0, 0], 1.0, xD, xL)
        assert len(pts) == 1
        p = pts[0]
        assert np.linalg.norm(r["pos"][q][0] - p) < 1e-4 * ext
        occ = _occlusion_closed_form(xD, p, xL, 1e-3)
        if occ is None:
            continue
        n[occ] += 1
        if occ:
            assert r["status"][q] == 5 and r["G"][q] == 0.0 and r["T"][q] == 0.0 and r["w"][q] == 0.0
        else:
            assert r["status"][q] == 0
            assert r["G"][q] == pytest.approx(CF.coddington_G([0, 0, 0], 1.0, xD, [0, 1, 0], xL, p), rel=1e-6)
    print(n)
    assert n[True] > 150 and n[False] > 500
    # the same walks without the rectangles: every OCCLUDED one converges (V is the only difference)
    s0 = O.OracleScene(W.config0(n_side=48, spp=4))
    r0 = s0.walks(np.nonzero(r["status"] == 5)[0], s0.opts(tol=1e-11, max_iters=40))
    assert (r0["status"] == 0).mean() > 0.99


def test_visibility_equals_brute_force_any_hit_cfg4():
    """configs[4] (cross-object occlusion between the sphere, the icosphere and the
    pool): the oracle's status of converged chains (CONVERGED vs OCCLUDED) equals a
    brute-force any-hit of every segment x_D -> x_1 -> ... -> x_k -> x_L against all
    surfaces (numpy Moller-Trumbore over every triangle, analytic sphere)."""
    w = W.config4(n_side=128, grid_n=64)
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks))
    pos, _, idx, _, _ = w.mesh_arrays()
    P = pos.astype(np.float64)
    v0, v1, v2 = P[idx[:, 0]], P[idx[:, 1]], P[idx[:, 2]]
    sph = [(np.asarray(f.center, np.float64), float(f.radius)) for f in w.surfaces if f.kind == W.SURF_SPHERE]
    eps = 1e-4 * s.extent
    sel = np.nonzero(np.isin(r["status"], (0, 5)))[0]
    n_occ = 0
    for q in sel:
        k = int(r["k"][q])
        pts = [w.xD[q // w.spp].astype(np.float64)] + [r["pos"][q][i] for i in range(k)] + [r["xL"][q]]
        occ = any(CF.any_hit_brute_force(pts[j], pts[j + 1], v0, v1, v2, sph, eps) for j in range(k + 1))
        assert occ == (r["status"][q] == 5), q
        n_occ += occ
    print(len(sel), n_occ)
    assert len(sel) > 100 and n_occ > 5
