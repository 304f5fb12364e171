// photons.cuh -- photon-based initial distribution p_0 (PAPER.md
// P:398 "reconstruct energy distributions from photons", "photon"
// initialization; reading R33).  One thread per photon: emission from a light,
// specular bounces (R with probability F at dielectrics, conductors R) traced
// with the scene BVH, fp64 positions and directions between fp32 traversals (as
// the deduction), landing on the receiver plane.  A landed photon with 1..6
// specular vertices is a sample record (x_D, x_L, w_D*, type, w = its power);
// the STree + vMF guide of iteration 0 is fitted from these records.
#pragma once

struct PhotonDev {
    int64_t n;             // N (power normalisation)
    uint64_t seed, base;
    double3 pp, pn;        // receiver plane point / unit normal
    int maxv;
    float eps;
};

__device__ __forceinline__ double fresnel_d(double ci, double e1, double e2) {
    ci = fabs(ci);
    double st2 = (e1 / e2) * (e1 / e2) * (1.0 - ci * ci);
    if (st2 >= 1.0) return 1.0;
    double ct = sqrt(1.0 - st2);
    double rs = (e1 * ci - e2 * ct) / (e1 * ci + e2 * ct);
    double rp = (e2 * ci - e1 * ct) / (e2 * ci + e1 * ct);
    return 0.5 * (rs * rs + rp * rp);
}

template <int W>
__global__ void k_photons(const DScene S, const PhotonDev P, int64_t first, int64_t count, mpg_guide_sample *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t wid = P.base + (uint64_t)(first + i);
        mpg_guide_sample rec;
        rec.xD[0] = rec.xD[1] = rec.xD[2] = 0.f;
        rec.xL[0] = rec.xL[1] = rec.xL[2] = 0.f;
        rec.omega[0] = rec.omega[1] = rec.omega[2] = 0.f;
        rec.w = 0.f;
        rec.type = -1;
        rec.pad = 0;
        // emission (purposes 8, 9)
        const uint4 r = rng_draw(P.seed, wid, 8u, 0u);
        const int li = S.n_light > 1 ? (int)uidx(r.z, (uint32_t)S.n_light) : 0;
        const DLight &L = S.light[li];
        const uint4 q = rng_draw(P.seed, wid, 9u, 0u);
        const double u1 = (double)u01(q.x), ph = 6.28318530717958647692 * (double)u01(q.y);
        float3 xLf;
        double phi;
        double3 d;
        if (L.kind == 1) {
            float a = FS(u01(r.x), 0.5f), b = FS(u01(r.y), 0.5f);
            xLf = f3(FA(L.pos.x, FA(FM(a, L.eu.x), FM(b, L.ev.x))), FA(L.pos.y, FA(FM(a, L.eu.y), FM(b, L.ev.y))),
                     FA(L.pos.z, FA(FM(a, L.eu.z), FM(b, L.ev.z))));
            double3 eu = d3f(L.eu), ev = d3f(L.ev);
            double3 nl = make_double3(eu.y * ev.z - eu.z * ev.y, eu.z * ev.x - eu.x * ev.z, eu.x * ev.y - eu.y * ev.x);
            double area = sqrt(ddot(nl, nl));
            nl = nl * (1.0 / area);
            phi = (double)L.emit * area * 3.14159265358979323846;
            double sg = copysign(1.0, nl.z), aa = -1.0 / (sg + nl.z), bb = nl.x * nl.y * aa;
            double3 b1 = make_double3(1.0 + sg * nl.x * nl.x * aa, sg * bb, -sg * nl.x);
            double3 b2 = make_double3(bb, sg + nl.y * nl.y * aa, -nl.y);
            double st = sqrt(u1), ct = sqrt(1.0 - u1);
            d = nl * ct + b1 * (st * cos(ph)) + b2 * (st * sin(ph));
        } else {
            xLf = L.pos;
            phi = 4.0 * 3.14159265358979323846 * (double)L.emit;
            double z = 1.0 - 2.0 * u1, st = sqrt(fmax(0.0, 1.0 - z * z));
            d = make_double3(st * cos(ph), z, st * sin(ph));
        }
        double w = (double)S.n_light * phi / (double)P.n;
        double3 o = d3f(xLf);
        double3 last = o;
        uint32_t bits = 0;
        int nv = 0;
        uint4 rt = make_uint4(0, 0, 0, 0);
        LaneStats ls = {0, 0, 0};
        for (;;) {
            Hit h;
            const bool hit = trace<W>(S, f3d(o), nrmz(f3d(d)), P.eps, 3.0e38f, false, false, h, ls);
            const double den = ddot(d, P.pn);
            const double tp = den < 0.0 ? ddot(P.pp - o, P.pn) / den : -1.0;
            if (tp > (double)P.eps && (!hit || tp < (double)h.t)) { // lands on the receiver plane
                if (nv >= 1) {
                    const float3 xD = f3d(o + d * tp);
                    const float3 v1 = f3d(last);
                    float dx = FS(v1.x, xD.x), dy = FS(v1.y, xD.y), dz = FS(v1.z, xD.z);
                    float l = __fsqrt_rn(FA(FA(FM(dx, dx), FM(dy, dy)), FM(dz, dz)));
                    rec.xD[0] = xD.x; rec.xD[1] = xD.y; rec.xD[2] = xD.z;
                    rec.xL[0] = xLf.x; rec.xL[1] = xLf.y; rec.xL[2] = xLf.z;
                    rec.omega[0] = FD(dx, l); rec.omega[1] = FD(dy, l); rec.omega[2] = FD(dz, l);
                    uint32_t tau = 0;
                    for (int j = 0; j < nv; j++) tau |= ((bits >> (nv - 1 - j)) & 1u) << j; // x_D order
                    rec.type = (1 << nv) - 2 + (int)tau;
                    rec.w = (float)w;
                }
                break;
            }
            if (!hit || nv == P.maxv) break;               // escaped, or longer than the guide's chains
            const DSurf &f = S.surf[h.surf];
            if (f.mat == 2) break;                         // absorbed by a diffuse occluder
            const double3 y = refine_hit(S, h.prim, h.surf, o, o + d, h.p);   // may move h.prim across a shared edge
            // normals in fp64 at the fp64 vertex (as the deduction, scatter_dir)
            const V3<double> ngd = geo_normalR<double>(S, h.prim, h.surf, y);
            V3<double> dna, dnb;
            const V3<double> z0 = mk3<double>(0.0, 0.0, 0.0);
            const V3<double> nsd = shadingR<double>(S, h.prim, h.surf, y, z0, z0, dna, dnb);
            double3 n = make_double3(nsd.x, nsd.y, nsd.z);
            n = n * rsqrt(ddot(n, n));
            const bool outside = ddot(d, make_double3(ngd.x, ngd.y, ngd.z)) < 0.0;
            if (ddot(d, n) > 0.0) n = n * -1.0;
            const double ci = -ddot(d, n);
            if (!(ci > 0.0)) break;
            uint32_t t = 0;
            // vertex nv owns word nv&3 of draw (10, nv>>2), whatever its material (R33)
            if ((nv & 3) == 0) rt = rng_draw(P.seed, wid, 10u, (uint32_t)(nv >> 2));
            if (f.mat == 0) {
                w *= (double)f.refl;
            } else {
                const double e1 = outside ? f.eta_out : f.eta_in, e2 = outside ? f.eta_in : f.eta_out;
                const double F = fresnel_d(ci, e1, e2);
                const uint32_t ru = (nv & 3) == 0 ? rt.x : (nv & 3) == 1 ? rt.y : (nv & 3) == 2 ? rt.z : rt.w;
                t = (double)u01(ru) >= F ? 1u : 0u;
                if (t) {
                    const double eta = e1 / e2;
                    const double k2 = 1.0 - eta * eta * (1.0 - ci * ci);
                    if (k2 < 0.0) break;
                    d = d * eta + n * (eta * ci - sqrt(k2));
                    d = d * rsqrt(ddot(d, d));
                }
            }
            if (!t) d = d + n * (2.0 * ci);
            bits |= t << nv;
            o = y;
            last = y;
            nv++;
        }
        out[i] = rec;
    }
}

extern "C" mpg_status mpg_trace_photons(const mpg_scene *scene, const mpg_photon_desc *pd, mpg_guide_sample *records,
                                        void *stream) {
    ARG_CHECK(scene && pd && (records || pd->n_photons == 0), "NULL argument");
    ARG_CHECK(pd->n_photons >= 0 && pd->max_vertices >= 1 && pd->max_vertices <= 6, "bad photon description");
    if (pd->n_photons == 0) return MPG_OK;
    PhotonDev P;
    P.n = pd->n_photons;
    P.seed = pd->seed;
    P.base = pd->photon_id_base;
    P.pp = make_double3(pd->plane_point[0], pd->plane_point[1], pd->plane_point[2]);
    double3 pn = make_double3(pd->plane_normal[0], pd->plane_normal[1], pd->plane_normal[2]);
    double l = std::sqrt(pn.x * pn.x + pn.y * pn.y + pn.z * pn.z);
    ARG_CHECK(l > 0.0, "zero plane normal");
    P.pn = make_double3(pn.x / l, pn.y / l, pn.z / l);
    P.maxv = pd->max_vertices;
    P.eps = pd->ray_eps > 0.f ? pd->ray_eps : 1e-4f * scene->d.extent;
    const int64_t n = pd->n_photons;
    int blocks = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
    COUNT_LAUNCH(1);
    if (scene->d.bvh_w == 4)
        k_photons<4><<<blocks, 128, 0, as_stream(stream)>>>(scene->d, P, 0, n, records);
    else
        k_photons<2><<<blocks, 128, 0, as_stream(stream)>>>(scene->d, P, 0, n, records);
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}
