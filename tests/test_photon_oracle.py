"""Pins of the oracle's photon tracer (photon-based p_0; R33).

A landed photon is a specular chain the emitter actually lights: its vertices
must be the admissible chain of (x_D, x_L) the closed forms give (Alhazen on
the mirror sphere, Snell on flat water), satisfy the manifold constraints
(C = 0), and carry the emitted power.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_12818_b200 import workloads as W
from tests import closed_forms as CF


def test_photons_on_the_mirror_sphere_hit_the_alhazen_point():
    w = W.config0(n_side=8, spp=1)
    s = O.OracleScene(w)
    rec, nv, verts, prims, surfs = s.trace_photons(20000, (0, -1.5, 0), (0, 1, 0))
    landed = nv >= 1
    assert landed.sum() > 100
    assert (nv[landed] == 1).all() and (rec["type"][landed] == 0).all()          # one R vertex
    sph = w.surfaces[0]
    for i in np.nonzero(landed)[0][:200]:
        xD, xL = rec["xD"][i].astype(np.float64), rec["xL"][i].astype(np.float64)
        pts = CF.alhazen_points(np.array(sph.center), sph.radius, xD, xL)
        d = min(np.linalg.norm(verts[i, 0] - p) for p in pts)
        assert d < 1e-5, (i, d)
        # w_D* points from x_D to the vertex
        om = verts[i, 0] - xD
        assert np.allclose(rec["omega"][i], om / np.linalg.norm(om), atol=1e-6)
    # power: isotropic point light (4 pi I) split over N photons; rho = 1 keeps it
    assert np.allclose(rec["w"][landed], 4 * np.pi / 20000, rtol=1e-6)
    # the fraction that hits the sphere is its solid angle from the light (1 - cos a)/2, sin a = r/d;
    # every hit reflects, those going down land
    hit_frac = (1 - np.sqrt(1 - (1 / 4.0) ** 2)) / 2
    assert landed.mean() < hit_frac + 4 * np.sqrt(hit_frac / 20000)


def test_photons_through_flat_water_follow_snell():
    w = W.config2(n_side=4, spp=1, flat=True, grid_n=16)
    s = O.OracleScene(w)
    rec, nv, verts, prims, surfs = s.trace_photons(4000, (0, -2, 0), (0, 1, 0), max_vertices=1)
    landed = nv == 1
    assert landed.sum() > 200
    assert (rec["type"][landed] == 1).all()                                         # T
    for i in np.nonzero(landed)[0][:200]:
        x1, _ = CF.snell_plane(rec["xD"][i], rec["xL"][i], 1.33, 1.0, 0.0)
        assert np.linalg.norm(verts[i, 0] - x1) < 2e-5
    # power: Lambertian unit square, radiance 1 -> pi; times (1 - F) survival is by choice, not weight
    assert np.allclose(rec["w"][landed], np.pi / 4000, rtol=1e-6)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg4"])
def test_photon_chains_satisfy_the_constraints(cfg):
    w = W.config1(n_side=4) if cfg == "cfg1" else W.config4(n_side=4, grid_n=32)
    s = O.OracleScene(w)
    rec, nv, verts, prims, surfs = s.trace_photons(6000, (0, -1.2 if cfg == "cfg1" else -2.0, 0), (0, 1, 0))
    landed = np.nonzero(nv >= 1)[0]
    assert len(landed) > 50
    worst = 0.0
    for i in landed[:300]:
        k = int(nv[i])
        tau = int(rec["type"][i]) - ((1 << k) - 2)
        ok, Cv, _ = s.constraint(k, tau, rec["xD"][i], rec["xL"][i], verts[i, :k], prims[i, :k], surfs[i, :k])
        assert ok
        worst = max(worst, np.abs(Cv).max())
    assert worst < 1e-4, worst


def _mirror_over_glass():
    """A downward-facing plane mirror (conductor) at y = 5 over a horizontal glass
    interface (eta 1.5 below) at y = 0, point light at (0, 4, 0): photons emitted
    upwards hit the conductor first, then the dielectric."""
    mirror = W.Surface(W.SURF_QUAD, W.MAT_CONDUCTOR, reflectance=1.0, origin=(-10.0, 5.0, -10.0),
                       edge_u=(20.0, 0.0, 0.0), edge_v=(0.0, 0.0, 20.0))
    glass = W.Surface(W.SURF_QUAD, W.MAT_DIELECTRIC, eta_in=1.5, eta_out=1.0, origin=(-10.0, 0.0, -10.0),
                      edge_u=(0.0, 0.0, 20.0), edge_v=(20.0, 0.0, 0.0))
    light = W.Light(W.LIGHT_POINT, 1.0, position=(0.0, 4.0, 0.0))
    xD, nD = W.receiver_grid(-1.0, 1.0, 2, -1.0)
    return W.Workload("mirror_over_glass", [mirror, glass], [light], xD, nD, 1, W.SeedSpec(W.SEED_CAP), W.WalkOpts())


def test_photon_RT_choice_after_a_conductor_vertex_follows_fresnel():
    """R33 / P:398: at every dielectric vertex a photon refracts with probability
    1 - F (exact Fresnel), also when an earlier vertex was a conductor (the R/T
    uniform of vertex v is word v&3 of draw (10, v>>2), whatever the materials).
    Count of landed light-order chains (conductor R, dielectric T) = N E[1 - F(cos)]
    over the upward emission directions that reach the glass, expectation by an
    independent numpy Monte Carlo of the same geometry."""
    w = _mirror_over_glass()
    s = O.OracleScene(w)
    n = 40000
    rec, nv, verts, prims, surfs = s.trace_photons(n, (0, -1.0, 0), (0, 1, 0))
    # type in x_D order: vertex 0 = the glass (T, bit 0), vertex 1 = the mirror (R): (1 << 2) - 2 + 0b01
    got = int(((nv == 2) & (rec["type"] == (1 << 2) - 2 + 1)).sum())
    rng = np.random.default_rng(123)
    m = 2_000_000
    z = rng.uniform(-1, 1, m)
    ph = rng.uniform(0, 2 * np.pi, m)
    st = np.sqrt(1 - z * z)
    d = np.stack([st * np.cos(ph), z, st * np.sin(ph)], 1)
    up = d[:, 1] > 0
    t1 = (5.0 - 4.0) / np.where(up, d[:, 1], 1.0)
    p1 = np.array([0.0, 4.0, 0.0]) + t1[:, None] * d                    # mirror hit
    t2 = 5.0 / np.where(up, d[:, 1], 1.0)                               # down to y = 0 after reflection
    p2 = p1 + t2[:, None] * d * np.array([1.0, -1.0, 1.0])
    ok = up & (np.abs(p1[:, 0]) < 10) & (np.abs(p1[:, 2]) < 10) & (np.abs(p2[:, 0]) < 10) & (np.abs(p2[:, 2]) < 10)
    cos = d[ok, 1]
    sint = np.sqrt(1 - cos ** 2) / 1.5
    ct = np.sqrt(1 - sint ** 2)
    rs = (cos - 1.5 * ct) / (cos + 1.5 * ct)
    rp = (1.5 * cos - ct) / (1.5 * cos + ct)
    p_T = (1 - 0.5 * (rs ** 2 + rp ** 2)).sum() / m
    exp = n * p_T
    print(got, exp)
    assert exp > 1000 and abs(got - exp) < 4 * np.sqrt(exp)
