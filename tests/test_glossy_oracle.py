"""Glossy chains via sampled offset normals (reading R37): pins of
the oracle.  Per walk, each chain vertex on a glossy surface (GGX alpha > 0) gets an offset normal
m = (a, b, 1) in its shading frame (s, t, n), drawn once per walk from D(m) cos(theta_m) and reused
by every trial; the chain must then satisfy h || m, i.e. C = (s.h - a n.h, t.h - b n.h) = 0.

Pins: the analytic Jacobian (with the exact derivative of the frame) equals central FD at admissible
glossy chains, Newton converges quadratically, the analytic GGT equals FD re-convergence, a glossy
plane mirror lands where an independent numpy root of the tilted reflection law puts it (with its
FD GGT), and alpha -> 0 recovers the specular chain (Alhazen point, Coddington G)."""
import numpy as np
import pytest
from scipy.optimize import fsolve

from oracle import oracle as O
from paper_2311_12818_b200 import workloads as W
from tests import closed_forms as CF


def walk_uv(w, walk_ids, k):
    """Offset uniforms of walks (reading R37): vertex i takes words 2(i&1), 2(i&1)+1 of Philox
    draw (walk id, purpose 11 + i//2, trial 0); u = (x >> 8) 2^-24."""
    out = np.zeros((len(walk_ids), k, 2))
    seed = w.opts.seed
    for j, wid in enumerate(np.asarray(walk_ids, np.uint64) + np.uint64(w.opts.walk_id_base)):
        for i in range(k):
            ctr = np.array([[int(wid) & 0xffffffff, int(wid) >> 32, 11 + (i >> 1), 0]], np.uint32)
            r = O.philox(ctr, (seed & 0xffffffff, seed >> 32))[0]
            out[j, i] = [(r[2 * (i & 1)] >> 8) * 2.0 ** -24, (r[2 * (i & 1) + 1] >> 8) * 2.0 ** -24]
    return out


def _glossy(which):
    return {"sphere": lambda: W.config0(16, 4, roughness=0.3),
            "glass_sphere": lambda: W.config1(16, 2, analytic=True, roughness=0.15),
            "icosphere": lambda: W.config1(24, 1, roughness=0.1)}[which]()


@pytest.mark.parametrize("which", ["sphere", "glass_sphere", "icosphere"])
def test_glossy_jacobian_matches_fd_at_admissible_chains(which):
    w = _glossy(which)
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks))
    idx = np.nonzero(r["status"] == 0)[0]
    assert len(idx) >= 5
    k, tau = w.seed.k, w.seed.tau
    uv = walk_uv(w, r["walk"][idx[:10]], k)
    worst = 0.0
    for j, q in enumerate(idx[:10]):
        O.set_offset_uv(uv[j])
        xD = w.xD[r["walk"][q] // w.spp].astype(np.float64)
        pos, prim, surf = r["pos"][q], r["prim"][q], r["surf"][q]
        ok, C0, J = s.constraint(k, tau, xD, r["xL"][q], pos, prim, surf)
        assert ok and np.abs(C0).max() < 1e-5            # the walk's own offsets: admissible
        for v_i in range(k):
            sg, tg = s.tangent_basis(prim[v_i], surf[v_i], pos[v_i])
            for c, v in enumerate((sg, tg)):
                h = 1e-6
                pp, pm = pos.copy(), pos.copy()
                pp[v_i] += h * v
                pm[v_i] -= h * v
                _, Cp, _ = s.constraint(k, tau, xD, r["xL"][q], pp, prim, surf)
                _, Cm, _ = s.constraint(k, tau, xD, r["xL"][q], pm, prim, surf)
                worst = max(worst, np.max(np.abs((Cp - Cm) / (2 * h) - J[:, 2 * v_i + c])) / max(1, np.abs(J).max()))
    O.set_offset_uv(None)
    assert worst < 1e-5, worst


def test_glossy_newton_converges_quadratically():
    w = _glossy("sphere")
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks), s.opts(tol=1e-12, max_iters=60))
    idx = np.nonzero(r["status"] == 0)[0]
    q = idx[0]
    O.set_offset_uv(walk_uv(w, [r["walk"][q]], 1)[0])
    xD = w.xD[r["walk"][q] // w.spp].astype(np.float64)
    p0 = r["pos"][q][0]
    sg, tg = s.tangent_basis(-1, 0, p0)
    res = []
    ds = np.geomspace(1e-2, 1e-4, 6)
    for d in ds:
        p = p0 + d * (sg + 0.5 * tg)
        p = p / np.linalg.norm(p)
        st, it, pos, prim, surf, hist = s.newton_chain(1, 0, xD, r["xL"][q], [p], [-1], [0], s.opts(max_iters=1, tol=0.0))
        res.append(hist[1] / hist[0] ** 2)
    O.set_offset_uv(None)
    slope = np.polyfit(np.log(ds), np.log(np.array(res) * ds ** 2), 1)[0]
    assert 1.8 <= slope <= 2.2, slope


@pytest.mark.parametrize("which", ["sphere", "glass_sphere", "icosphere"])
def test_glossy_ggt_analytic_equals_fd_reconvergence(which):
    w = _glossy(which)
    w.opts.tol, w.opts.max_iters = 1e-12, 60
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks))
    idx = np.nonzero(r["status"] == 0)[0]
    k, tau = w.seed.k, w.seed.tau
    uv = walk_uv(w, r["walk"][idx[:12]], k)
    checked = 0
    for j, q in enumerate(idx[:12]):
        O.set_offset_uv(uv[j])
        xD = w.xD[r["walk"][q] // w.spp]
        a = s.ggt(k, tau, xD, w.nD[0], r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q], method=0)
        f1 = s.ggt(k, tau, xD, w.nD[0], r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q], method=1, delta=2e-6)
        f2 = s.ggt(k, tau, xD, w.nD[0], r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q], method=1, delta=1e-6)
        if f1 < 0 or f2 < 0:
            continue
        checked += 1
        assert f1 == pytest.approx(f2, rel=1e-5) and a == pytest.approx(f2, rel=1e-5)
        assert a == pytest.approx(r["G"][q], rel=1e-10)     # the walk's G used the same offsets
    O.set_offset_uv(None)
    assert checked >= 5


def _duff(n):
    sign = np.copysign(1.0, n[2])
    a = -1.0 / (sign + n[2])
    b = n[0] * n[1] * a
    return np.array([1 + sign * n[0] ** 2 * a, sign * b, -sign * n[0]]), np.array([b, sign + n[1] ** 2 * a, -n[1]])


def test_glossy_plane_mirror_tilted_reflection_law():
    """A glossy plane mirror z = 0 with a fixed offset: the chain is where ray optics about the
    tilted normal n' = normalize(n + a s + b t) sends x_D to x_L (numpy root of the reflection
    law, independent of the oracle's Newton), and G equals numpy FD of that root map."""
    alpha = 0.4
    quad = W.Surface(W.SURF_QUAD, W.MAT_CONDUCTOR, reflectance=1.0, origin=(-5.0, -5.0, 0.0), edge_u=(10.0, 0.0, 0.0),
                     edge_v=(0.0, 10.0, 0.0), roughness=alpha)
    light = W.Light(W.LIGHT_POINT, 1.0, position=(2.0, 0.5, 1.5))
    xD = np.array([0.0, 0.0, 1.0])
    w = W.Workload("glossy_plane", [quad], [light], xD[None].astype(np.float32), np.array([[0, 0, 1]], np.float32), 1,
                   W.SeedSpec(W.SEED_CAP), W.WalkOpts())
    s = O.OracleScene(w)
    for uv in ([0.3, 0.7], [0.05, 0.2], [0.6, 0.95]):
        O.set_offset_uv(np.array([uv]))
        tt = alpha * np.sqrt(uv[0] / (1 - uv[0]))
        a, b = tt * np.cos(2 * np.pi * uv[1]), tt * np.sin(2 * np.pi * uv[1])
        n = np.array([0.0, 0.0, 1.0])
        sv, tv = _duff(n)
        npr = n + a * sv + b * tv
        npr /= np.linalg.norm(npr)

        def law(pxy, xL):
            p = np.array([pxy[0], pxy[1], 0.0])
            h = CF.nz(CF.nz(xD - p) + CF.nz(xL - p))
            return np.cross(h, npr)[:2]

        xL = np.array([2.0, 0.5, 1.5])
        p = fsolve(law, [1.0, 0.2], args=(xL,), xtol=1e-14)
        out = s.walk_from_target(xD, [0, 0, 1], xL, [p[0] + 0.05, p[1] - 0.03, 0.0], opts=s.opts(tol=1e-12, max_iters=60))
        assert out["status"] == 0
        assert np.allclose(out["pos"][0][:2], p, atol=1e-9) and abs(out["pos"][0][2]) < 1e-12
        # G by numpy FD of the root map x_L -> p -> w_D (point light: axes orthogonal to x_L - p)
        e1, e2 = _duff(CF.nz(xL - np.array([p[0], p[1], 0.0])))
        dw = []
        for ax in (e1, e2):
            ws = []
            for sg in (1, -1):
                q = fsolve(law, p, args=(xL + sg * 1e-6 * ax,), xtol=1e-14)
                ws.append(CF.nz(np.array([q[0], q[1], 0.0]) - xD))
            dw.append((ws[0] - ws[1]) / 2e-6)
        wD = CF.nz(np.array([p[0], p[1], 0.0]) - xD)
        f1, f2 = _duff(wD)
        M = np.array([[f1 @ dw[0], f1 @ dw[1]], [f2 @ dw[0], f2 @ dw[1]]])
        G_fd = abs(wD[2]) * abs(np.linalg.det(M))
        assert out["G"] == pytest.approx(G_fd, rel=1e-5)
    O.set_offset_uv(None)


def test_glossy_alpha_to_zero_is_the_specular_chain():
    """alpha -> 0: the offset vanishes and every converged chain is the specular one
    (Alhazen point, Coddington G) although the glossy code path (exact frame derivative) runs."""
    w = W.config0(24, 4, roughness=1e-12)
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks), s.opts(tol=1e-11, max_iters=40))
    idx = np.nonzero(r["status"] == 0)[0]
    assert len(idx) > 200
    for q in idx[::5]:
        xD = w.xD[r["walk"][q] // w.spp].astype(np.float64)
        pts = CF.alhazen_points([0, 0, 0], 1.0, xD, r["xL"][q])
        assert np.linalg.norm(r["pos"][q][0] - pts[0]) < 1e-8
        assert r["G"][q] == pytest.approx(CF.coddington_G([0, 0, 0], 1.0, xD, [0, 1, 0], r["xL"][q], pts[0]), rel=1e-7)


def test_glossy_walks_differ_from_specular_and_keep_their_offsets():
    """With alpha > 0 the converged chains move off the specular solution (the offset is in
    effect), and each satisfies the constraint with its own walk's offsets (trials reuse them)."""
    w = _glossy("sphere")
    s = O.OracleScene(w)
    r = s.walks(np.arange(w.n_walks))
    idx = np.nonzero(r["status"] == 0)[0]
    moved = 0
    uv = walk_uv(w, r["walk"][idx[:40]], 1)
    for j, q in enumerate(idx[:40]):
        xD = w.xD[r["walk"][q] // w.spp].astype(np.float64)
        pts = CF.alhazen_points([0, 0, 0], 1.0, xD, r["xL"][q])
        moved += bool(pts) and np.linalg.norm(r["pos"][q][0] - pts[0]) > 1e-3
        O.set_offset_uv(uv[j])
        ok, C0, _ = s.constraint(1, 0, xD, r["xL"][q], r["pos"][q], r["prim"][q], r["surf"][q])
        assert np.abs(C0).max() < 1e-5
    O.set_offset_uv(None)
    assert moved > 20
