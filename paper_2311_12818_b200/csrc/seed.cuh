// seed.cuh -- light samples and seed-chain targets (device), shared by the
// seed kernel (primary walks, trial 0) and the walk kernel (trials t >= 1).
//
// P:395-406 (initialization: x_1 uniform on specular surfaces)
// (Eq. 8), P:501-512 (Eq. 13 defensive mixture, alpha = 1/2), P:337 (x_L by
// uniform emitter sampling).  All arithmetic that decides a seed is fp32
// without contraction (R23), so the oracle's plain C float code draws the
// same seeds; discrete choices are integer-exact (R2, R20).
#pragma once
#include "device_common.cuh"

struct SeedCtx {
    int mode, surf_id, k;
    uint32_t tau;
    uint64_t seed;
    // guide (MPG_SEED_GUIDE_UV)
    float gox, goz, gex, gez;
    int cells_x, cells_y, bins_x, bins_y;
    float uvox, uvoz, uvsx, uvsz, uv_y;
    const uint64_t *prefix; // [cells][bins] inclusive prefix of W'
    // typed direction guide (MPG_SEED_GUIDE_DIR, configs[4], R22)
    const uint64_t *n_prefix;    // [cells][6]
    const uint64_t *type_prefix; // [cells][126]
    const uint32_t *dir_prefix;  // [cells][126][bins]
    // STree + vMF guide (MPG_SEED_GUIDE_STREE): n_prefix /
    // type_prefix above are then per leaf
    int root_ref;                           // >= 0 inner node, < 0: ~leaf
    const int4 *nodes;                      // (split as bits, axis, child0, child1)
    const int *grp_off;                     // [leaves][127] lobe offsets of (leaf, type) groups
    const unsigned long long *lobe_prefix;  // [lobes] inclusive per-group prefix of W_i
    const float4 *lobe_mu;                  // [lobes] mu (xyz), kappa (w)
    const int *leaf_own;                    // [leaves] own (non-copy) samples per leaf (R36)
    int selective;                          // MPG_FLAG_SELECTIVE: empty leaf -> INACTIVE
};

// one seed draw: the deduction ray x_D -> tgt gives x_1 (Eq. 6); n = chain
// length; bits = tau (learned / fixed type) or per-vertex R/T choices of the
// initializer (learned = false); Pn = P(n)
struct SeedRes {
    float3 tgt;
    int bin, n;
    uint32_t bits;
    bool learned;
    float Pn;
};

__device__ __forceinline__ uint64_t mulhi_u64(uint32_t x, uint64_t S) { // floor(x*S/2^32), exact
    uint64_t X = x;
    return X * (S >> 32) + ((X * (S & 0xffffffffull)) >> 32);
}

__device__ __forceinline__ int seed_cell(const SeedCtx &g, float3 xD) {
    int cx = (int)floorf(FD(FM(FS(xD.x, g.gox), (float)g.cells_x), g.gex));
    int cz = (int)floorf(FD(FM(FS(xD.z, g.goz), (float)g.cells_y), g.gez));
    cx = min(max(cx, 0), g.cells_x - 1);
    cz = min(max(cz, 0), g.cells_y - 1);
    return cz * g.cells_x + cx;
}

// x_L (purpose 0, trial 0) (R15); returns its pdf
__device__ __forceinline__ float sample_light(const DScene &S, uint64_t seed, uint64_t wid, float3 &xL, int &lid) {
    uint4 r = rng_draw(seed, wid, 0u, 0u);
    int li = S.n_light > 1 ? (int)uidx(r.z, (uint32_t)S.n_light) : 0;
    const DLight &L = S.light[li];
    lid = li;
    if (L.kind == 1) {
        float a = u01(r.x) - 0.5f, b = u01(r.y) - 0.5f;
        xL = f3(FA(L.pos.x, FA(FM(a, L.eu.x), FM(b, L.ev.x))), FA(L.pos.y, FA(FM(a, L.eu.y), FM(b, L.ev.y))),
                FA(L.pos.z, FA(FM(a, L.eu.z), FM(b, L.ev.z))));
    } else {
        xL = L.pos;
    }
    return L.pdf;
}

__device__ __forceinline__ void onb_exact(float3 n, float3 &b1, float3 &b2) {
    float sign = copysignf(1.0f, n.z);
    float a = FD(-1.0f, FA(sign, n.z));
    float b = FM(FM(n.x, n.y), a);
    b1 = f3(FA(1.0f, FM(FM(FM(sign, n.x), n.x), a)), FM(sign, b), FM(-sign, n.x));
    b2 = f3(b, FA(sign, FM(FM(n.y, n.y), a)), -n.y);
}

// Seed target for (walk, trial): the deduction ray x_D -> target gives x_1
// (Eq. 6).  Returns false if no seed could be drawn (SEED_FAIL), with bin = -3 if
// the walk is inactive (selective activation, R36).
// w_D ~ vMF(mu, kappa) (Eq. 12) by the inverse CDF of cos(theta) (R31)
__device__ __forceinline__ float3 vmf_dir(float4 m, float u1, float u2) {
    float kap = m.w;
    float xi = FS(1.0f, u1);
    float e2k = expf(FM(-2.0f, kap));
    float ct = FA(1.0f, FD(logf(FA(xi, FM(FS(1.0f, xi), e2k))), kap));
    ct = fminf(fmaxf(ct, -1.0f), 1.0f);
    float st2 = FS(1.0f, FM(ct, ct));
    float st = __fsqrt_rn(st2 > 0.0f ? st2 : 0.0f);
    float phi = FM(6.28318530717958647692f, u2);
    float cp = cosf(phi), sp = sinf(phi);
    float3 b1, b2;
    float3 mu = f3(m.x, m.y, m.z);
    onb_exact(mu, b1, b2);
    return f3(FA(FM(ct, mu.x), FM(st, FA(FM(cp, b1.x), FM(sp, b2.x)))),
              FA(FM(ct, mu.y), FM(st, FA(FM(cp, b1.y), FM(sp, b2.y)))),
              FA(FM(ct, mu.z), FM(st, FA(FM(cp, b1.z), FM(sp, b2.z)))));
}

__device__ __forceinline__ float canon0(float x) { return __fadd_rn(x, 0.0f); } // -0 -> +0 (R28)

// leaf of the STree containing (x_D, x_L) (R28).  Out of line, like the lobe draw
// below: seed_target is inlined into k_walk, whose instruction-cache footprint is a
// measured limiter (configs[4] +4 % with these paths inlined)
__device__ __noinline__ int stree_leaf(const SeedCtx &g, float3 xD, float3 xL) {
    float p[6] = {canon0(xD.x), canon0(xD.y), canon0(xD.z), canon0(xL.x), canon0(xL.y), canon0(xL.z)};
    int ref = g.root_ref;
    int guard = 0;
    while (ref >= 0) {
        MPG_CHECK(++guard <= 64);
        int4 nd = __ldg(g.nodes + ref);
        float v = p[0];
#pragma unroll
        for (int a = 1; a < 6; a++) v = nd.y == a ? p[a] : v;
        ref = v < __int_as_float(nd.x) ? nd.z : nd.w;
    }
    return ~ref;
}

// mode 4, learned branch: lobe i of group (leaf, type) by the integer CDF of W_i, then
// w_D ~ vMF(mu_i, kappa_i) (Eq. 12, R30-R31); returns the deduction target x_D + w_D
__device__ __noinline__ float3 stree_lobe_target(const SeedCtx &g, int grp, uint32_t rw, uint64_t wid, uint32_t trial,
                                                 float3 xD, int &bin) {
    const int *go = g.grp_off + grp;
    int glo = __ldg(go), ghi = __ldg(go + 1);
    MPG_CHECK(glo < ghi);
    uint64_t Sl = __ldg(g.lobe_prefix + ghi - 1);
    uint64_t tl = mulhi_u64(rw, Sl);
    int lo2 = glo, hi2 = ghi - 1; // upper_bound over the group
    while (lo2 < hi2) {
        int mid = (lo2 + hi2) >> 1;
        if ((uint64_t)__ldg(g.lobe_prefix + mid) > tl) hi2 = mid;
        else lo2 = mid + 1;
    }
    bin = lo2;
    uint4 r2 = rng_draw(g.seed, wid, 2u, trial);
    float3 om = vmf_dir(__ldg(g.lobe_mu + lo2), u01(r2.x), u01(r2.y));
    return f3(FA(xD.x, om.x), FA(xD.y, om.y), FA(xD.z, om.z));
}

// stage / stage_cell: the seed kernel's copy of one cell's prefix table in shared memory
// (north_star: "CDF tables staged in shared memory"), used when the walk's cell is that cell
__device__ MPG_COLD bool seed_target(const DScene &S, const SeedCtx &g, uint64_t wid, uint32_t trial,
                                            float3 xD, float3 xL, SeedRes &sr,
                                            const unsigned long long *stage = nullptr, int stage_cell = -1) {
    float3 &tgt = sr.tgt;
    int &bin = sr.bin;
    bin = -1;
    sr.n = g.k;
    sr.bits = g.tau;
    sr.learned = true;
    sr.Pn = 1.0f;
    if (g.mode == 0) { // uniform on the cap of a sphere visible from x_D
        const DSurf &f = S.surf[g.surf_id];
        float dx = FS(xD.x, f.center.x), dy = FS(xD.y, f.center.y), dz = FS(xD.z, f.center.z);
        float L = __fsqrt_rn(FA(FA(FM(dx, dx), FM(dy, dy)), FM(dz, dz)));
        float3 a = f3(FD(dx, L), FD(dy, L), FD(dz, L));
        float cmin = FD(f.radius, L);
        uint4 r = rng_draw(g.seed, wid, 2u, trial);
        float u1 = u01(r.x), u2 = u01(r.y);
        float ct = FS(1.0f, FM(u1, FS(1.0f, cmin)));
        float st2 = FS(1.0f, FM(ct, ct));
        float st = __fsqrt_rn(st2 > 0.0f ? st2 : 0.0f);
        float phi = FM(6.28318530717958647692f, u2);
        float cp = cosf(phi), sp = sinf(phi);
        float3 b1, b2;
        onb_exact(a, b1, b2);
        float ddx = FA(FM(ct, a.x), FM(st, FA(FM(cp, b1.x), FM(sp, b2.x))));
        float ddy = FA(FM(ct, a.y), FM(st, FA(FM(cp, b1.y), FM(sp, b2.y))));
        float ddz = FA(FM(ct, a.z), FM(st, FA(FM(cp, b1.z), FM(sp, b2.z))));
        tgt = f3(FA(f.center.x, FM(f.radius, ddx)), FA(f.center.y, FM(f.radius, ddy)),
                 FA(f.center.z, FM(f.radius, ddz)));
        return true;
    }
    if (g.mode == 1) { // triangle uniform by count among front-facing, <= 32 rejection draws
        const DSurf &f = S.surf[g.surf_id];
        int tri = -1;
        float3 v0, e1, e2;
        for (uint32_t rr = 0; rr < 32u; rr++) {
            uint4 r = rng_draw(g.seed, wid, 16u + rr, trial);
            int t = f.tri_begin + (int)uidx(r.x, (uint32_t)f.tri_count);
            int4 ix = __ldg(S.oidx + t);
            float3 p0 = xyz(__ldg(S.vpos + ix.x)), p1 = xyz(__ldg(S.vpos + ix.y)), p2 = xyz(__ldg(S.vpos + ix.z));
            float3 a = f3(FS(p1.x, p0.x), FS(p1.y, p0.y), FS(p1.z, p0.z));
            float3 b = f3(FS(p2.x, p0.x), FS(p2.y, p0.y), FS(p2.z, p0.z));
            float ngx = FS(FM(a.y, b.z), FM(a.z, b.y));
            float ngy = FS(FM(a.z, b.x), FM(a.x, b.z));
            float ngz = FS(FM(a.x, b.y), FM(a.y, b.x));
            float dd = FA(FA(FM(FS(xD.x, p0.x), ngx), FM(FS(xD.y, p0.y), ngy)), FM(FS(xD.z, p0.z), ngz));
            if (dd > 0.0f) { tri = t; v0 = p0; e1 = a; e2 = b; break; }
        }
        if (tri < 0) return false;
        bin = tri;
        uint4 r = rng_draw(g.seed, wid, 2u, trial);
        float u1 = u01(r.x), u2 = u01(r.y);
        float sq = __fsqrt_rn(u1);
        float c1 = FM(sq, FS(1.0f, u2)), c2 = FM(sq, u2);
        tgt = f3(FA(v0.x, FA(FM(c1, e1.x), FM(c2, e2.x))), FA(v0.y, FA(FM(c1, e1.y), FM(c2, e2.y))),
                 FA(v0.z, FA(FM(c1, e1.z), FM(c2, e2.z))));
        return true;
    }
    if (g.mode == 2) { // guided bin over the surface (u,v): integer CDF of W' (R20)
        int nb = g.bins_x * g.bins_y;
        const int cell = seed_cell(g, xD);
        const uint64_t *pf = g.prefix + (size_t)cell * nb;
        uint4 r = rng_draw(g.seed, wid, 1u, trial);
        uint64_t x = r.x;
        int lo = 0, hi = nb - 1; // upper_bound: first b with prefix[b] > t
        if (stage && cell == stage_cell) {   // the table staged in shared memory
            const uint64_t S_ = stage[nb - 1];
            const uint64_t t = x * (S_ >> 32) + ((x * (S_ & 0xffffffffull)) >> 32); // floor(x*S/2^32)
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if ((uint64_t)stage[mid] > t) hi = mid;
                else lo = mid + 1;
            }
        } else {
            const uint64_t S_ = __ldg((const unsigned long long *)pf + nb - 1);
            const uint64_t t = x * (S_ >> 32) + ((x * (S_ & 0xffffffffull)) >> 32);
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if ((uint64_t)__ldg((const unsigned long long *)pf + mid) > t) hi = mid;
                else lo = mid + 1;
            }
        }
        bin = lo;
        int bx = lo % g.bins_x, by = lo / g.bins_x;
        uint4 r2 = rng_draw(g.seed, wid, 2u, trial);
        float u = FD(FA((float)bx, u01(r2.x)), (float)g.bins_x);
        float v = FD(FA((float)by, u01(r2.y)), (float)g.bins_y);
        tgt = f3(FA(g.uvox, FM(u, g.uvsx)), g.uv_y, FA(g.uvoz, FM(v, g.uvsz)));
        return true;
    }
    if (g.mode == 3 || g.mode == 4) { // configs[4]: n ~ 1/2 P_0 + 1/2 P_e, then one-sample MIS for (w_D, tau)
        // (R22); mode 4: P_e from the STree leaf of (x_D, x_L), w_D from its vMF mixture (R28-R31)
        int c = g.mode == 3 ? seed_cell(g, xD) : stree_leaf(g, xD, xL);
        // selective activation (R36): no own sample in the leaf -> path tracing
        if (g.mode == 4 && g.selective && __ldg(g.leaf_own + c) == 0) { bin = -3; return false; }
        const unsigned long long *npf = (const unsigned long long *)g.n_prefix + (size_t)c * 6;
        uint4 r0 = rng_draw(g.seed, wid, 1u, 0u); // n is reused by every trial
        uint64_t S6 = __ldg(npf + 5);
        uint64_t t = mulhi_u64(r0.x, S6);
        int n = 0;
        while ((uint64_t)__ldg(npf + n) <= t) n++;
        uint64_t lo = n > 0 ? (uint64_t)__ldg(npf + n - 1) : 0ull;
        sr.Pn = (float)((double)((uint64_t)__ldg(npf + n) - lo) / (double)S6);
        n += 1;
        sr.n = n;
        uint4 r = rng_draw(g.seed, wid, 1u, trial);
        int g0 = (1 << n) - 2, gn = 1 << n;
        const unsigned long long *tpf = (const unsigned long long *)g.type_prefix + (size_t)c * 126 + g0;
        uint64_t Wg = __ldg(tpf + gn - 1);
        float u, v;
        if (Wg > 0 && (r.y >> 31)) {
            uint64_t tt = mulhi_u64(r.z, Wg);
            int m = 0;
            while ((uint64_t)__ldg(tpf + m) <= tt) m++;
            sr.bits = (uint32_t)m;
            sr.learned = true;
            if (g.mode == 4) { // lobe ~ W_i, then w_D ~ vMF(mu_i, kappa_i) (Eq. 12)
                tgt = stree_lobe_target(g, c * 127 + g0 + m, r.w, wid, trial, xD, bin);
                return true;
            }
            int nb = g.bins_x * g.bins_y;
            const uint32_t *dpf = g.dir_prefix + ((size_t)c * 126 + g0 + m) * nb;
            uint64_t Sd = __ldg(dpf + nb - 1);
            uint64_t td = mulhi_u64(r.w, Sd);
            int lo2 = 0, hi2 = nb - 1;
            while (lo2 < hi2) {
                int mid = (lo2 + hi2) >> 1;
                if ((uint64_t)__ldg(dpf + mid) > td) hi2 = mid;
                else lo2 = mid + 1;
            }
            bin = lo2;
            uint4 r2 = rng_draw(g.seed, wid, 2u, trial);
            u = FD(FA((float)(lo2 % g.bins_x), u01(r2.x)), (float)g.bins_x);
            v = FD(FA((float)(lo2 / g.bins_x), u01(r2.y)), (float)g.bins_y);
        } else {
            uint4 r3 = rng_draw(g.seed, wid, 3u, trial);
            u = u01(r3.x);
            v = u01(r3.y);
            sr.learned = false;
            sr.bits = r3.z;
        }
        // equal-area hemisphere about +y: u = cos(theta), v = (phi + pi)/(2 pi)
        float st2 = FS(1.0f, FM(u, u));
        float st = __fsqrt_rn(st2 > 0.0f ? st2 : 0.0f);
        float phi = FS(FM(6.28318530717958647692f, v), 3.14159265358979323846f);
        float cp = cosf(phi), sp = sinf(phi);
        tgt = f3(FA(xD.x, FM(st, cp)), FA(xD.y, u), FA(xD.z, FM(st, sp)));
        return true;
    }
    return false;
}
