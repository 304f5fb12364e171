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
