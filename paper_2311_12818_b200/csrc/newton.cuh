// newton.cuh -- the manifold-walk Newton system, generic over the scalar type R
// of the Jacobian / frame / step arithmetic (R = float: default product path;
// R = double: MPG_FLAG_NEWTON_F64).  Vertex positions and the residual C are
// always fp64 (R24).
//
// Per vertex i with a = x_{i-1}, p = x_i, b = x_{i+1} (x_0 = x_D, x_{k+1} = x_L):
//   w_i = (a-p)/|a-p|, w_o = (b-p)/|b-p| (away from p, R1),
//   h~ = eta_i w_i + eta_o w_o, h = h~/|h~|, (s,t) = ONB(n_s) (R3), C_i = (s.h, t.h).
// Blocks (displacement v on a tangent plane, R4):
//   L: dh = P_h(eta_i P_i v)   U: dh = P_h(eta_o P_o v)
//   D: dh = P_h(-eta_i P_i v - eta_o P_o v), minus (h.n)(s.dn) for the frame (R3)
// with P_i v = (v - w_i(w_i.v))/l_i, P_h u = (u - h(h.u))/|h~|.  Block-Thomas
// elimination is fused into the sweep: only D'^-1_i, U_i, r'_i survive.
#pragma once
#include "device_common.cuh"

#ifndef MPG_ROLL_DC
#define MPG_ROLL_DC 0
#endif
template <typename R> struct V3 {
    R x, y, z;
};
template <typename R> __device__ __forceinline__ V3<R> mk3(R x, R y, R z) { return {x, y, z}; }
template <typename R> __device__ __forceinline__ V3<R> fromf(float3 a) { return {(R)a.x, (R)a.y, (R)a.z}; }
template <typename R> __device__ __forceinline__ V3<R> fromd(double3 a) { return {(R)a.x, (R)a.y, (R)a.z}; }
template <typename R> __device__ __forceinline__ float3 tof(V3<R> a) { return make_float3((float)a.x, (float)a.y, (float)a.z); }
template <typename R> __device__ __forceinline__ double3 tod(V3<R> a) { return make_double3(a.x, a.y, a.z); }
template <typename R> __device__ __forceinline__ V3<R> operator+(V3<R> a, V3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <typename R> __device__ __forceinline__ V3<R> operator-(V3<R> a, V3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <typename R> __device__ __forceinline__ V3<R> operator-(V3<R> a) { return {-a.x, -a.y, -a.z}; }
template <typename R> __device__ __forceinline__ V3<R> operator*(V3<R> a, R s) { return {a.x * s, a.y * s, a.z * s}; }
template <typename R> __device__ __forceinline__ R dotR(V3<R> a, V3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <typename R> __device__ __forceinline__ V3<R> crossR(V3<R> a, V3<R> b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ float rsq(float v) { return rsqrtf(v); }
__device__ __forceinline__ double rsq(double v) { return rsqrt(v); }
template <typename R> __device__ __forceinline__ R lenR(V3<R> a) { return sqrt(dotR(a, a)); }
template <typename R> __device__ __forceinline__ V3<R> nrmR(V3<R> a) { return a * rsq(dotR(a, a)); }

template <typename R> __device__ __forceinline__ void onbR(V3<R> n, V3<R> &b1, V3<R> &b2) {
    R sign = copysign((R)1, n.z);
    R a = (R)-1 / (sign + n.z);
    R b = n.x * n.y * a;
    b1 = {(R)1 + sign * n.x * n.x * a, sign * b, -sign * n.x};
    b2 = {b, sign + n.y * n.y * a, -n.y};
}
// derivative of that basis for a change dn of n (glossy vertices: with an offset normal the
// frame's twist does not drop out of the constraint at the solution, R37)
template <typename R> __device__ __forceinline__ void onb_dR(V3<R> n, V3<R> dn, V3<R> &d1, V3<R> &d2) {
    R sign = copysign((R)1, n.z);
    R a = (R)-1 / (sign + n.z);
    R da = a * a * dn.z;
    R db = (dn.x * n.y + n.x * dn.y) * a + n.x * n.y * da;
    d1 = {sign * ((R)2 * n.x * dn.x * a + n.x * n.x * da), sign * db, -sign * dn.x};
    d2 = {db, (R)2 * n.y * dn.y * a + n.y * n.y * da, -dn.y};
}

// Glossy chains (R37): offset slopes (a, b) of chain vertex i, i.e. the offset
// normal m = (a, b, 1) in the vertex's shading frame, GGX(alpha) by D(m) cos(theta_m):
// tan(theta_m) = alpha sqrt(u1 / (1 - u1)), phi = 2 pi u2, with (u1, u2) = words 2(i&1),
// 2(i&1)+1 of Philox (walk, purpose 11 + i/2, trial 0) -- once per walk, reused by trials
__device__ __forceinline__ void glossy_slopes(const DScene &S, int surf, uint64_t seed, uint64_t wid, int i,
                                              double &a, double &b) {
    a = b = 0.0;
    const float al = S.surf[surf].rough;
    if (!(al > 0.0f)) return;
    const uint4 r = rng_draw(seed, wid, 11u + (uint32_t)(i >> 1), 0u);
    const double u1 = (double)u01((i & 1) ? r.z : r.x), u2 = (double)u01((i & 1) ? r.w : r.y);
    const double tt = (double)al * sqrt(u1 / (1.0 - u1));
    const double ph = 6.28318530717958647692 * u2;
    a = tt * cos(ph);
    b = tt * sin(ph);
}

// geometric normal (outward, R9)
template <typename R> __device__ __forceinline__ V3<R> geo_normalR(const DScene &S, int prim, int surf, double3 p) {
    if (prim >= 0) {
        V3<R> v0 = fromf<R>(xyz(__ldg(S.tpos + TSTRIDE * prim))), v1 = fromf<R>(xyz(__ldg(S.tpos + TSTRIDE * prim + 1))),
              v2 = fromf<R>(xyz(__ldg(S.tpos + TSTRIDE * prim + 2)));
        return nrmR(crossR(v1 - v0, v2 - v0));
    }
    const DSurf &f = S.surf[surf];
    if (f.kind == 0) return nrmR(fromd<R>(make_double3(p.x - f.center.x, p.y - f.center.y, p.z - f.center.z)));
    return fromf<R>(f.nq);
}

// shading normal and its derivatives along tangent vectors a, b (Phong / sphere / quad)
template <typename R>
__device__ __forceinline__ V3<R> shadingR(const DScene &S, int prim, int surf, double3 p, V3<R> a, V3<R> b,
                                          V3<R> &dna, V3<R> &dnb) {
    if (prim >= 0) {
        float3 fv0 = xyz(__ldg(S.tpos + TSTRIDE * prim));
        V3<R> v0 = fromf<R>(fv0), v1 = fromf<R>(xyz(__ldg(S.tpos + TSTRIDE * prim + 1))),
              v2 = fromf<R>(xyz(__ldg(S.tpos + TSTRIDE * prim + 2)));
        V3<R> n0 = fromf<R>(xyz(__ldg(S.tnrm + 3 * prim))), n1 = fromf<R>(xyz(__ldg(S.tnrm + 3 * prim + 1))),
              n2 = fromf<R>(xyz(__ldg(S.tnrm + 3 * prim + 2)));
        V3<R> e1 = v1 - v0, e2 = v2 - v0;
        V3<R> Ng = crossR(e1, e2);
        R inv = (R)1 / dotR(Ng, Ng);
        V3<R> g1 = crossR(e2, Ng) * inv, g2 = crossR(Ng, e1) * inv;
        V3<R> r = fromd<R>(make_double3(p.x - fv0.x, p.y - fv0.y, p.z - fv0.z));
        R c1 = dotR(r, g1), c2 = dotR(r, g2), c0 = (R)1 - c1 - c2;
        V3<R> nt = n0 * c0 + n1 * c1 + n2 * c2;
        R il = rsq(dotR(nt, nt));
        V3<R> n = nt * il;
        V3<R> d1 = n1 - n0, d2 = n2 - n0;
        V3<R> ta = d1 * dotR(a, g1) + d2 * dotR(a, g2);
        V3<R> tb = d1 * dotR(b, g1) + d2 * dotR(b, g2);
        dna = (ta - n * dotR(n, ta)) * il;
        dnb = (tb - n * dotR(n, tb)) * il;
        return n;
    }
    const DSurf &f = S.surf[surf];
    if (f.kind == 0) {
        V3<R> rr = fromd<R>(make_double3(p.x - f.center.x, p.y - f.center.y, p.z - f.center.z));
        R il = rsq(dotR(rr, rr));
        V3<R> n = rr * il;
        dna = (a - n * dotR(n, a)) * il;
        dnb = (b - n * dotR(n, b)) * il;
        return n;
    }
    dna = mk3<R>(0, 0, 0);
    dnb = dna;
    return fromf<R>(f.nq);
}

template <typename R> __device__ __forceinline__ R fresnelR(R ci, R eta1, R eta2) {
    ci = fabs(ci);
    R e = eta1 / eta2;
    R st2 = e * e * ((R)1 - ci * ci);
    if (st2 >= (R)1) return (R)1;
    R ct = sqrt((R)1 - st2);
    R rs = (eta1 * ci - eta2 * ct) / (eta1 * ci + eta2 * ct);
    R rp = (eta2 * ci - eta1 * ct) / (eta2 * ci + eta1 * ct);
    return (R)0.5 * (rs * rs + rp * rp);
}

template <typename R, bool GL> struct VTermR {
    V3<R> wi, wo, h, s, t, n;
    R li, lo, ei, eo, hl, hn;
    R oa, ob;        // offset slopes (glossy, R37)
    bool glossy;
    double c0, c1;
};

// residual always fp64 from fp64 positions (R24); the rest in R
template <typename R, bool GL>
__device__ __forceinline__ bool vtermR(double3 a, double3 p, double3 b, V3<R> ng, V3<R> n, const DSurf &f, bool isT,
                                       VTermR<R, GL> &v, double oa = 0.0, double ob = 0.0) {
    double ax = a.x - p.x, ay = a.y - p.y, az = a.z - p.z;
    double bx = b.x - p.x, by = b.y - p.y, bz = b.z - p.z;
    double la2 = ax * ax + ay * ay + az * az, lb2 = bx * bx + by * by + bz * bz;
    if (!(la2 > 0.0) || !(lb2 > 0.0)) return false;
    double ia = rsqrt(la2), ib = rsqrt(lb2);
    ax *= ia; ay *= ia; az *= ia;
    bx *= ib; by *= ib; bz *= ib;
    v.li = (R)(la2 * ia);
    v.lo = (R)(lb2 * ib);
    v.wi = mk3<R>((R)ax, (R)ay, (R)az);
    v.wo = mk3<R>((R)bx, (R)by, (R)bz);
    if (isT) {
        bool out = dotR(v.wi, ng) > (R)0;
        v.ei = out ? (R)f.eta_out : (R)f.eta_in;
        v.eo = out ? (R)f.eta_in : (R)f.eta_out;
    } else {
        v.ei = v.eo = (R)1;
    }
    double hx = (double)v.ei * ax + (double)v.eo * bx, hy = (double)v.ei * ay + (double)v.eo * by,
           hz = (double)v.ei * az + (double)v.eo * bz;
    double hl2 = hx * hx + hy * hy + hz * hz;
    if (!(hl2 > 0.0) || !isfinite(hl2)) return false;
    double ih = rsqrt(hl2);
    hx *= ih; hy *= ih; hz *= ih;
    v.hl = (R)(hl2 * ih);
    v.h = mk3<R>((R)hx, (R)hy, (R)hz);
    onbR(n, v.s, v.t);
    v.c0 = (double)v.s.x * hx + (double)v.s.y * hy + (double)v.s.z * hz;
    v.c1 = (double)v.t.x * hx + (double)v.t.y * hy + (double)v.t.z * hz;
    v.hn = dotR(v.h, n);
    if constexpr (GL) {
    v.n = n;
    v.glossy = f.rough > 0.0f;
    v.oa = (R)oa;
    v.ob = (R)ob;
    if (v.glossy) {  // h || m = (a, b, 1) in (s, t, n): C = (s.h - a n.h, t.h - b n.h) (R37)
        const double hn = (double)n.x * hx + (double)n.y * hy + (double)n.z * hz;
        v.c0 -= oa * hn;
        v.c1 -= ob * hn;
    }
    }
    return true;
}

// dC along a neighbour displacement (L, U, D_L blocks)
template <typename R, bool GL>
__device__ __forceinline__ void dC_nbR(const VTermR<R, GL> &v, V3<R> w, R l, R eta, V3<R> dir, R &o0, R &o1) {
    V3<R> u = (dir - w * dotR(w, dir)) * (eta / l);
    V3<R> dh = (u - v.h * dotR(v.h, u)) * ((R)1 / v.hl);
    o0 = dotR(v.s, dh);
    o1 = dotR(v.t, dh);
    if constexpr (GL) {
        if (v.glossy) {
            const R ndh = dotR(v.n, dh);
            o0 -= v.oa * ndh;
            o1 -= v.ob * ndh;
        }
    }
}
// dC along the vertex's own displacement (D block; minimal-rotation frame, R3)
template <typename R, bool GL>
__device__ __forceinline__ void dC_selfR(const VTermR<R, GL> &v, V3<R> dir, V3<R> dn, R &o0, R &o1) {
    V3<R> u = (dir - v.wi * dotR(v.wi, dir)) * (-v.ei / v.li) - (dir - v.wo * dotR(v.wo, dir)) * (v.eo / v.lo);
    V3<R> dh = (u - v.h * dotR(v.h, u)) * ((R)1 / v.hl);
    if constexpr (GL) {
        if (v.glossy) {  // exact frame derivative and the offset terms (R37)
            V3<R> ds, dt;
            onb_dR(v.n, dn, ds, dt);
            const R dhn = dotR(dn, v.h) + dotR(v.n, dh);
            o0 = dotR(ds, v.h) + dotR(v.s, dh) - v.oa * dhn;
            o1 = dotR(dt, v.h) + dotR(v.t, dh) - v.ob * dhn;
            return;
        }
    }
    o0 = dotR(v.s, dh) - v.hn * dotR(v.s, dn);
    o1 = dotR(v.t, dh) - v.hn * dotR(v.t, dn);
}

// Forward sweep (constraint + blocks + block-Thomas) and, if not converged,
// back substitution into world-space steps dq.  Returns 0 step, 1 converged,
// 2 degenerate; `singular` flags a singular pivot (G is then 0 at convergence).
template <int KMAX, typename R, bool GL>
__device__ __forceinline__ int newton_system(const DScene &S, uint64_t seed, uint64_t wid, int k, uint32_t tau,
                                             float3 xD, float3 xL,
                                             const double3 (&x)[KMAX], const int (&prim)[KMAX],
                                             const int (&surf)[KMAX], float tol, R (&Di)[KMAX][4], R (&Ub)[KMAX][4],
                                             V3<R> (&sg)[KMAX], V3<R> (&tg)[KMAX], V3<R> (&dq)[KMAX],
                                             bool &singular, float &cmax_out) {
    R rp[KMAX][2];
    bool degen = false;
    singular = false;
    double cmax = 0.0;
#pragma unroll
    for (int i = 0; i < KMAX; i++) {
        if (i >= k) break;
        onbR(geo_normalR<R>(S, prim[i], surf[i], x[i]), sg[i], tg[i]);
    }
    // rolled: one copy of the per-vertex body keeps the hot code small (ncu: 37% of the
    // persistent kernel's stall samples were instruction-fetch stalls with it unrolled)
#pragma unroll 1
    for (int i = 0; i < KMAX; i++) {
        if (i >= k) break;
        const double3 xi = rget(x, i);
        const int pi = rget(prim, i), si = rget(surf, i);
        const V3<R> sgi = rget(sg, i), tgi = rget(tg, i);
        double3 a = i == 0 ? d3f(xD) : rget(x, i > 0 ? i - 1 : 0);
        double3 b = i == k - 1 ? d3f(xL) : rget(x, i + 1 < KMAX ? i + 1 : i);
        const DSurf &f = S.surf[si];
        V3<R> dna, dnb;
        V3<R> n = shadingR<R>(S, pi, si, xi, sgi, tgi, dna, dnb);
        VTermR<R, GL> v;
        double oa = 0.0, ob = 0.0;
        if constexpr (GL) glossy_slopes(S, si, seed, wid, i, oa, ob);
        if (!vtermR<R, GL>(a, xi, b, crossR(sgi, tgi), n, f, (tau >> i) & 1u, v, oa, ob)) { degen = true; break; }
        cmax = fmax(cmax, fmax(fabs(v.c0), fabs(v.c1)));
        // the two tangent directions (MPG_ROLL_DC: in a rolled loop, one copy of the block
        // code; A/B in DESIGN.md §4)
        R D00, D10, D01, D11;
#if MPG_ROLL_DC
#pragma unroll 1
#else
#pragma unroll
#endif
        for (int c = 0; c < 2; c++) {
            R o0, o1;
            dC_selfR(v, c ? tgi : sgi, c ? dnb : dna, o0, o1);
            if (c == 0) { D00 = o0; D10 = o1; } else { D01 = o0; D11 = o1; }
        }
        R r0 = (R)(-v.c0), r1 = (R)(-v.c1);
        if (i > 0) {
            const int j = i > 0 ? i - 1 : 0;
            R l00, l10, l01, l11;
            const V3<R> sgj = rget(sg, j), tgj = rget(tg, j);
#if MPG_ROLL_DC
#pragma unroll 1
#else
#pragma unroll
#endif
            for (int c = 0; c < 2; c++) {
                R o0, o1;
                dC_nbR(v, v.wi, v.li, v.ei, c ? tgj : sgj, o0, o1);
                if (c == 0) { l00 = o0; l10 = o1; } else { l01 = o0; l11 = o1; }
            }
            const R d0 = rget2(Di, j, 0), d1 = rget2(Di, j, 1), d2 = rget2(Di, j, 2), d3 = rget2(Di, j, 3);
            const R u0 = rget2(Ub, j, 0), u1 = rget2(Ub, j, 1), u2 = rget2(Ub, j, 2), u3 = rget2(Ub, j, 3);
            R M00 = l00 * d0 + l01 * d2, M01 = l00 * d1 + l01 * d3;
            R M10 = l10 * d0 + l11 * d2, M11 = l10 * d1 + l11 * d3;
            D00 -= M00 * u0 + M01 * u2;
            D01 -= M00 * u1 + M01 * u3;
            D10 -= M10 * u0 + M11 * u2;
            D11 -= M10 * u1 + M11 * u3;
            const R p0 = rget2(rp, j, 0), p1 = rget2(rp, j, 1);
            r0 -= M00 * p0 + M01 * p1;
            r1 -= M10 * p0 + M11 * p1;
        }
        if (i < k - 1) {
            const int j = i + 1 < KMAX ? i + 1 : i;
            R u00, u10, u01, u11;
            const V3<R> sgj = rget(sg, j), tgj = rget(tg, j);
#if MPG_ROLL_DC
#pragma unroll 1
#else
#pragma unroll
#endif
            for (int c = 0; c < 2; c++) {
                R o0, o1;
                dC_nbR(v, v.wo, v.lo, v.eo, c ? tgj : sgj, o0, o1);
                if (c == 0) { u00 = o0; u10 = o1; } else { u01 = o0; u11 = o1; }
            }
            rset2(Ub, i, 0, u00); rset2(Ub, i, 1, u01); rset2(Ub, i, 2, u10); rset2(Ub, i, 3, u11);
        }
        R det = D00 * D11 - D01 * D10;
        if (!(det != (R)0) || !isfinite(det)) singular = true;
        R id = (R)1 / det;
        rset2(Di, i, 0, D11 * id); rset2(Di, i, 1, -D01 * id); rset2(Di, i, 2, -D10 * id); rset2(Di, i, 3, D00 * id);
        rset2(rp, i, 0, r0); rset2(rp, i, 1, r1);
    }
    cmax_out = (float)cmax;
    if (degen || !isfinite(cmax)) return 2;
    if (cmax < (double)tol) return 1;
    if (singular) return 2;
    R n0 = 0, n1 = 0; // Delta_{i+1}
#pragma unroll
    for (int i = KMAX - 1; i >= 0; i--) {
        if (i > k - 1) continue;
        R r0 = rp[i][0], r1 = rp[i][1];
        if (i < k - 1) {
            r0 -= Ub[i][0] * n0 + Ub[i][1] * n1;
            r1 -= Ub[i][2] * n0 + Ub[i][3] * n1;
        }
        R a0 = Di[i][0] * r0 + Di[i][1] * r1;
        R a1 = Di[i][2] * r0 + Di[i][3] * r1;
        if (!isfinite(a0) || !isfinite(a1)) return 2;
        dq[i] = sg[i] * a0 + tg[i] * a1;
        n0 = a0; n1 = a1;
    }
    return 0;
}

// sides (R8), kappa (R12) and the light-side block D_L at a converged chain
template <int KMAX, typename R, bool GL>
__device__ MPG_COLD bool post_sweep(const DScene &S, uint64_t seed, uint64_t wid, const DLight &L, int k, uint32_t tau,
                                           float3 xD,
                                           float3 xL, const double3 (&x)[KMAX], const int (&prim)[KMAX],
                                           const int (&surf)[KMAX], bool want_kappa, float &kappa, R (&DL)[4]) {
    R kap = 1, etaD = 1, etaL = 1;
#pragma unroll 1
    for (int i = 0; i < KMAX; i++) {
        if (i >= k) break;
        const double3 xi = rget(x, i);
        const int pi = rget(prim, i), si = rget(surf, i);
        double3 a = i == 0 ? d3f(xD) : rget(x, i > 0 ? i - 1 : 0);
        double3 b = i == k - 1 ? d3f(xL) : rget(x, i + 1 < KMAX ? i + 1 : i);
        const DSurf &f = S.surf[si];
        V3<R> ng = geo_normalR<R>(S, pi, si, xi);
        R di = dotR(fromd<R>(a - xi), ng), dd = dotR(fromd<R>(b - xi), ng);
        bool isT = (tau >> i) & 1u;
        if (isT ? !(di * dd < (R)0) : !(di * dd > (R)0)) return false;
        if (!want_kappa) continue;
        V3<R> z = mk3<R>(0, 0, 0), dna, dnb;
        V3<R> n = shadingR<R>(S, pi, si, xi, z, z, dna, dnb);
        double oa = 0.0, ob = 0.0;
        if constexpr (GL) glossy_slopes(S, si, seed, wid, i, oa, ob);
        bool oi = di > (R)0, oo = dd > (R)0;
        R e_wi = oi ? (R)f.eta_out : (R)f.eta_in, e_wo = oo ? (R)f.eta_out : (R)f.eta_in;
        if (i == 0) etaD = e_wi;
        if (i == k - 1) {
            etaL = e_wo;
            VTermR<R, GL> v;
            if (!vtermR<R, GL>(a, xi, b, ng, n, f, isT, v, oa, ob)) { DL[0] = DL[1] = DL[2] = DL[3] = 0; }
            else {
                V3<R> l1, l2;
                if (L.kind == 1) { l1 = fromf<R>(L.l1); l2 = fromf<R>(L.l2); }
                else onbR(nrmR(fromd<R>(d3f(xL) - xi)), l1, l2);
                dC_nbR(v, v.wo, v.lo, v.eo, l1, DL[0], DL[2]);
                dC_nbR(v, v.wo, v.lo, v.eo, l2, DL[1], DL[3]);
            }
        }
        if (f.mat == 0) kap *= (R)f.refl;
        else {
            R e_other = oi ? (R)f.eta_in : (R)f.eta_out;
            V3<R> wi = nrmR(fromd<R>(a - xi));
            V3<R> nm = n;
            if (GL && f.rough > 0.0f) {  // Fresnel at the micro-normal (offset normal, R37)
                V3<R> s, t;
                onbR(n, s, t);
                nm = nrmR(n + s * (R)oa + t * (R)ob);
            }
            R F = fresnelR<R>(dotR(wi, nm), e_wi, e_other);
            kap *= isT ? ((R)1 - F) : F;
        }
    }
    kappa = (float)(kap * (etaD / etaL) * (etaD / etaL));
    return true;
}

// analytic GGT: back-substitute J Y = -[0..0; D_L] with the stored D'^-1, U (R11)
template <int KMAX, typename R>
__device__ MPG_COLD float ggt_from_blocks(int k, float3 xD, float3 nD, const double3 (&x)[KMAX],
                                                 const R (&Di)[KMAX][4], const R (&Ub)[KMAX][4],
                                                 const V3<R> (&sg)[KMAX], const V3<R> (&tg)[KMAX],
                                                 const R (&DL)[4]) {
    R y00 = 0, y01 = 0, y10 = 0, y11 = 0; // Y_{i+1}
#pragma unroll
    for (int i = KMAX - 1; i >= 0; i--) {
        if (i > k - 1) continue;
        R b00, b01, b10, b11;
        if (i == k - 1) { b00 = -DL[0]; b01 = -DL[1]; b10 = -DL[2]; b11 = -DL[3]; }
        else {
            b00 = -(Ub[i][0] * y00 + Ub[i][1] * y10);
            b01 = -(Ub[i][0] * y01 + Ub[i][1] * y11);
            b10 = -(Ub[i][2] * y00 + Ub[i][3] * y10);
            b11 = -(Ub[i][2] * y01 + Ub[i][3] * y11);
        }
        R n00 = Di[i][0] * b00 + Di[i][1] * b10, n01 = Di[i][0] * b01 + Di[i][1] * b11;
        R n10 = Di[i][2] * b00 + Di[i][3] * b10, n11 = Di[i][2] * b01 + Di[i][3] * b11;
        y00 = n00; y01 = n01; y10 = n10; y11 = n11;
    }
    V3<R> r = fromd<R>(x[0] - d3f(xD));
    R rl = lenR(r);
    V3<R> w = r * ((R)1 / rl);
    V3<R> e1, e2;
    onbR(w, e1, e2);
    V3<R> dx0 = sg[0] * y00 + tg[0] * y10, dx1 = sg[0] * y01 + tg[0] * y11;
    V3<R> dw0 = (dx0 - w * dotR(w, dx0)) * ((R)1 / rl), dw1 = (dx1 - w * dotR(w, dx1)) * ((R)1 / rl);
    R M00 = dotR(e1, dw0), M01 = dotR(e1, dw1), M10 = dotR(e2, dw0), M11 = dotR(e2, dw1);
    R G = fabs(dotR(fromf<R>(nD), w)) * fabs(M00 * M11 - M01 * M10);
    return isfinite(G) ? (float)G : 0.0f;
}
