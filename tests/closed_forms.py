"""Closed-form solutions used to pin the oracle (tests only).

Each function is an independent derivation (numpy, fp64) of a quantity the
paper's method must reproduce; none of them calls oracle/ or the CUDA path.
"""
import numpy as np


def nz(v):
    return v / np.linalg.norm(v)


def _roots_scan(f, lo, hi, n=20000, iters=80, fvec=None):
    xs = np.linspace(lo, hi, n + 1)
    fs = fvec(xs) if fvec is not None else np.array([f(x) for x in xs])
    roots = []
    for i in range(n):
        a, b, fa, fb = xs[i], xs[i + 1], fs[i], fs[i + 1]
        if not (np.isfinite(fa) and np.isfinite(fb)):
            continue
        if fa == 0.0:
            roots.append(a)
            continue
        if fa * fb < 0:
            for _ in range(iters):
                m = 0.5 * (a + b)
                fm = f(m)
                if not np.isfinite(fm):
                    break
                if fa * fm <= 0:
                    b, fb = m, fm
                else:
                    a, fa = m, fm
            roots.append(0.5 * (a + b))
    return roots


def _plane_axes(c, xD, xL):
    e1 = nz(xD - c)
    v = xL - c
    vp = v - e1 * np.dot(e1, v)
    if np.linalg.norm(vp) < 1e-12:
        vp = np.cross(e1, [1.0, 0.0, 0.0])
        if np.linalg.norm(vp) < 1e-6:
            vp = np.cross(e1, [0.0, 0.0, 1.0])
    return e1, nz(vp)


def alhazen_points(c, R, xD, xL):
    """Reflection points on a mirror sphere (Alhazen's problem), in-plane 1D roots
    of t.(w_D + w_L) = 0 on the great circle through c, x_D, x_L, keeping only
    points seen from both ends (n.(x_D-p) > 0 and n.(x_L-p) > 0)."""
    c, xD, xL = (np.asarray(a, np.float64) for a in (c, xD, xL))
    e1, e2 = _plane_axes(c, xD, xL)

    def f(phi):
        p = c + R * (np.cos(phi) * e1 + np.sin(phi) * e2)
        t = -np.sin(phi) * e1 + np.cos(phi) * e2
        return np.dot(nz(xD - p), t) + np.dot(nz(xL - p), t)

    def fv(phi):
        p = c + R * (np.cos(phi)[:, None] * e1 + np.sin(phi)[:, None] * e2)
        t = -np.sin(phi)[:, None] * e1 + np.cos(phi)[:, None] * e2
        a = xD - p
        b = xL - p
        a /= np.linalg.norm(a, axis=1, keepdims=True)
        b /= np.linalg.norm(b, axis=1, keepdims=True)
        return (a * t).sum(1) + (b * t).sum(1)

    out = []
    for phi in _roots_scan(f, -np.pi, np.pi, 4000, fvec=fv):
        p = c + R * (np.cos(phi) * e1 + np.sin(phi) * e2)
        n = (p - c) / R
        if np.dot(n, xD - p) > 0 and np.dot(n, xL - p) > 0:
            out.append(p)
    return out


def coddington_G(c, R, xD, nD, xL, p):
    """GGT of a point light reflected by a convex sphere mirror (Coddington
    equations for the tangential/sagittal virtual focal distances)."""
    c, xD, nD, xL, p = (np.asarray(a, np.float64) for a in (c, xD, nD, xL, p))
    n = (p - c) / R
    s = np.linalg.norm(xL - p)
    d = np.linalg.norm(xD - p)
    cos = np.dot(n, nz(xL - p))
    at = 1.0 / (1.0 / s + 2.0 / (R * cos))
    as_ = 1.0 / (1.0 / s + 2.0 * cos / R)
    cosD = abs(np.dot(nD, nz(p - xD)))
    return cosD * at * as_ / (s * s * (d + at) * (d + as_))


def _refract(d, n, eta1, eta2):
    if np.dot(d, n) > 0:
        n = -n
    ci = -np.dot(d, n)
    eta = eta1 / eta2
    k = 1.0 - eta * eta * (1.0 - ci * ci)
    if k < 0:
        return None
    return nz(eta * d + (eta * ci - np.sqrt(k)) * n)


def tt_sphere_chains(c, R, eta, xD, xL, near=None, width=0.02):
    """All in-plane TT chains through a glass sphere: x_1 on the great circle of
    the plane (c, x_D, x_L), refract in, chord, refract out, direction to x_L.
    `near` (a point) restricts the scan to +-width rad around its angle (for
    grazing chains, whose visible interval is narrower than the global scan step).
    Returns list of (x1, x2)."""
    c, xD, xL = (np.asarray(a, np.float64) for a in (c, xD, xL))
    e1, e2 = _plane_axes(c, xD, xL)
    nrm = np.cross(e1, e2)

    def trace(phi):
        p1 = c + R * (np.cos(phi) * e1 + np.sin(phi) * e2)
        n1 = (p1 - c) / R
        d = nz(p1 - xD)
        if np.dot(n1, xD - p1) <= 0:
            return None
        d2 = _refract(d, n1, 1.0, eta)
        if d2 is None:
            return None
        t = -2.0 * np.dot(d2, p1 - c)
        p2 = p1 + t * d2
        n2 = (p2 - c) / R
        d3 = _refract(d2, n2, eta, 1.0)
        if d3 is None:
            return None
        return p1, p2, d3

    def f(phi):
        r = trace(phi)
        if r is None:
            return np.nan
        p1, p2, d3 = r
        u = nz(xL - p2)
        if np.dot(d3, u) <= 0:
            return np.nan
        return np.dot(np.cross(d3, u), nrm)

    out = []
    lo, hi, n = -np.pi, np.pi, 8000
    if near is not None:
        q = np.asarray(near, np.float64) - c
        ph = np.arctan2(np.dot(q, e2), np.dot(q, e1))
        lo, hi, n = ph - width, ph + width, 2000
    for phi in _roots_scan(f, lo, hi, n):
        r = trace(phi)
        if r is not None:
            out.append((r[0], r[1]))
    return out


def snell_plane(xD, xL, eta1, eta2, y_surf=0.0):
    """Refraction point on the plane y=y_surf for x_D below (medium eta1) and x_L
    above (eta2): h1 tan(t1) + h2 tan(t2) = rho, eta1 sin t1 = eta2 sin t2.
    Returns (x1, G) with G the closed-form GGT for a horizontal light plane
    (G = cos t1 sin t1 / (rho drho/dt1))."""
    xD, xL = np.asarray(xD, np.float64), np.asarray(xL, np.float64)
    h1, h2 = y_surf - xD[1], xL[1] - y_surf
    dvec = np.array([xL[0] - xD[0], 0.0, xL[2] - xD[2]])
    rho = np.linalg.norm(dvec)
    tmax = np.arcsin(min(1.0, eta2 / eta1)) if eta1 > eta2 else 0.5 * np.pi

    def t2_of(t1):
        return np.arcsin(eta1 * np.sin(t1) / eta2)

    def F(t1):
        return h1 * np.tan(t1) + h2 * np.tan(t2_of(t1)) - rho

    a, b = 0.0, tmax * (1 - 1e-15)
    for _ in range(200):
        m = 0.5 * (a + b)
        if F(m) > 0:
            b = m
        else:
            a = m
    t1 = 0.5 * (a + b)
    t2 = t2_of(t1)
    u = dvec / rho if rho > 0 else np.array([1.0, 0.0, 0.0])
    x1 = xD + u * h1 * np.tan(t1) + np.array([0.0, h1, 0.0])
    drho = h1 / np.cos(t1) ** 2 + h2 / np.cos(t2) ** 2 * (eta1 * np.cos(t1)) / (eta2 * np.cos(t2))
    G = np.cos(t1) * np.sin(t1) / (rho * drho)
    return x1, G


def snell_layers(xD, xL, ys, etas, with_G=False):
    """Refraction points of the straight-up chain from x_D through horizontal
    interfaces y = ys[0] < ys[1] < ... to x_L; etas[i] is the index of the
    medium below ys[i] (etas[-1] the medium above the last interface).
    Snell's invariant p = eta sin(t) is the same in every layer, so the lateral
    offset is rho = sum_i h_i p / sqrt(eta_i^2 - p^2) (layer heights h_i);
    p is found by bisection (rho is increasing in p).  Returns [len(ys), 3], or
    with `with_G` also (G, kappa): G = d omega_L / dA_D for a point light at x_L
    in a medium of index 1 over a horizontal receiver,
    G = p / (cos t_L rho drho/dp), drho/dp = sum_i h_i eta_i^2 / (eta_i^2 - p^2)^(3/2),
    and kappa = prod over interfaces of (1 - F), F the unpolarised Fresnel
    reflectance (Hecht, Optics, §4.6.2) at that interface's angles."""
    xD, xL = np.asarray(xD, np.float64), np.asarray(xL, np.float64)
    yy = np.concatenate([[xD[1]], np.asarray(ys, np.float64), [xL[1]]])
    h = np.diff(yy)
    eta = np.asarray(etas, np.float64)
    assert np.all(h > 0) and len(eta) == len(h)
    dvec = np.array([xL[0] - xD[0], 0.0, xL[2] - xD[2]])
    rho = np.linalg.norm(dvec)
    pmax = eta.min()

    def offsets(p):
        return h * p / np.sqrt(eta * eta - p * p)

    a, b = 0.0, pmax * (1 - 1e-15)
    for _ in range(200):
        m = 0.5 * (a + b)
        if offsets(m).sum() > rho:
            b = m
        else:
            a = m
    p = 0.5 * (a + b)
    off = np.cumsum(offsets(p))[:-1]
    u = dvec / rho if rho > 0 else np.array([1.0, 0.0, 0.0])
    pts = np.array([xD + u * o + np.array([0.0, y - xD[1], 0.0]) for o, y in zip(off, ys)])
    if not with_G:
        return pts
    assert eta[-1] == 1.0
    drho = (h * eta * eta / (eta * eta - p * p) ** 1.5).sum()
    G = p / (np.sqrt(1.0 - p * p) * rho * drho)
    kappa = 1.0
    for e1, e2 in zip(eta[:-1], eta[1:]):
        ci, ct = np.sqrt(1 - (p / e1) ** 2), np.sqrt(1 - (p / e2) ** 2)
        rs = (e1 * ci - e2 * ct) / (e1 * ci + e2 * ct)
        rp = (e2 * ci - e1 * ct) / (e2 * ci + e1 * ct)
        kappa *= 1.0 - 0.5 * (rs * rs + rp * rp)
    return pts, G, kappa


def mirror_sphere_G(c, R, xD, nD, xL, p, light_normal=None):
    """GGT of a k = 1 reflection off a sphere mirror: the point-light form
    (coddington_G) times cos t_L at an area light of normal `light_normal`."""
    G = coddington_G(c, R, xD, nD, xL, p)
    if light_normal is not None:
        G *= abs(np.dot(nz(np.asarray(p, np.float64) - np.asarray(xL, np.float64)), light_normal))
    return G


def segment_hits_rect(a, b, rect, margin):
    """Does the open segment a -> b cross the axis-aligned horizontal rectangle
    rect = (origin, edge_u, edge_v) (edges along +x and +z, y constant)?  Returns
    True / False, or None when the crossing lies within `margin` of the rectangle's
    border (too close to call in floating point)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    o, u, v = (np.asarray(x, np.float64) for x in rect)
    y = o[1]
    if (a[1] - y) * (b[1] - y) >= 0:
        return False
    t = (y - a[1]) / (b[1] - a[1])
    p = a + t * (b - a)
    dx = min(p[0] - o[0], o[0] + u[0] - p[0])
    dz = min(p[2] - o[2], o[2] + v[2] - p[2])
    d = min(dx, dz)                     # > 0 inside, < 0 outside
    if abs(d) < margin:
        return None
    return bool(d > 0)


def any_hit_brute_force(a, b, tri_v0, tri_v1, tri_v2, spheres=(), eps=0.0):
    """Any intersection of the segment a -> b with t in (eps, |b-a| - eps) against
    every triangle (Moller-Trumbore over all of them, numpy fp64) and analytic
    spheres (c, R): the visibility V of Eq. 2 by brute force."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = b - a
    L = np.linalg.norm(d)
    d = d / L
    for c, R in spheres:
        oc = a - np.asarray(c, np.float64)
        bb = np.dot(oc, d)
        disc = bb * bb - (np.dot(oc, oc) - R * R)
        if disc >= 0:
            for t in (-bb - np.sqrt(disc), -bb + np.sqrt(disc)):
                if eps < t < L - eps:
                    return True
    if len(tri_v0) == 0:
        return False
    e1 = tri_v1 - tri_v0
    e2 = tri_v2 - tri_v0
    p = np.cross(d, e2)
    det = np.einsum("ij,ij->i", e1, p)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / det
        tv = a - tri_v0
        u = np.einsum("ij,ij->i", tv, p) * inv
        q = np.cross(tv, e1)
        v = (q @ d) * inv
        t = np.einsum("ij,ij->i", e2, q) * inv
    hit = (det != 0) & (u >= 0) & (v >= 0) & (u + v <= 1) & (t > eps) & (t < L - eps)
    return bool(hit.any())
