// device_common.cuh -- fp32 vector math, Philox4x32-10, scene records, ray
// intersection and BVH traversal for the sm_100a manifold-walk kernels.
//
// Everything here is the product path (no oracle code is shared).  Readings
// "Rn" refer to DESIGN.md §3; "P:n" to PAPER.md lines.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define MPG_FULL 0xffffffffu
// MPG_CHECKS=1: a bounds-checked build (device-side traps on out-of-range indices in the
// traversal stack, the trial ring / entry table, chain outputs and STree lookups).  It is
// the memory-error check of this repo: compute-sanitizer is closed on the GPU pool
// (profiles/r2_bounds_checks.log).  Off in the product build.
#ifndef MPG_CHECKS
#define MPG_CHECKS 0
#endif
#if MPG_CHECKS
#include <cstdio>
#define MPG_CHECK(cond)                                                                        \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("MPG_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                 \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define MPG_CHECK(cond) ((void)0)
#endif
// end-of-attempt / seeding helpers (__noinline__ measured slower than inlined:
// 3.3 KB stack frame, configs[1,3])
#ifndef MPG_COLD
#define MPG_COLD __forceinline__
#endif

// ----------------------------------------------------------------------------
// float3 helpers (contraction allowed: this is the Newton / traversal math)
// ----------------------------------------------------------------------------
__device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__device__ __forceinline__ float3 xyz(float4 a) { return make_float3(a.x, a.y, a.z); }
__device__ __forceinline__ float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ float3 operator-(float3 a) { return f3(-a.x, -a.y, -a.z); }
__device__ __forceinline__ float3 operator*(float3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float3 operator*(float s, float3 a) { return f3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float dot(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float3 cross(float3 a, float3 b) {
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float len(float3 a) { return sqrtf(dot(a, a)); }
__device__ __forceinline__ float3 nrmz(float3 a) { return a * rsqrtf(dot(a, a)); }
__device__ __forceinline__ float comp(float3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }

// fp64 points: chain vertex positions are kept in fp64 (see walk.cuh, R24)
__device__ __forceinline__ double3 d3f(float3 a) { return make_double3(a.x, a.y, a.z); }
__device__ __forceinline__ float3 f3d(double3 a) { return make_float3((float)a.x, (float)a.y, (float)a.z); }
__device__ __forceinline__ double3 operator+(double3 a, double3 b) { return make_double3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ double3 operator-(double3 a, double3 b) { return make_double3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double3 operator*(double3 a, double s) { return make_double3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ double ddot(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// Orthonormal basis of a unit vector (Duff et al. 2017); any basis is valid for
// the constraint frame and the step parameterization (R3, R4).
__device__ __forceinline__ void onb(float3 n, float3 &b1, float3 &b2) {
    float sign = copysignf(1.0f, n.z);
    float a = -1.0f / (sign + n.z);
    float b = n.x * n.y * a;
    b1 = f3(1.0f + sign * n.x * n.x * a, sign * b, -sign * n.x);
    b2 = f3(b, sign + n.y * n.y * a, -n.y);
}

// ----------------------------------------------------------------------------
// exact fp32 helpers for the seed path (R23): these intrinsics are never
// contracted into FMAs, so seeds match the oracle's plain C float arithmetic.
// ----------------------------------------------------------------------------
#define FM(a, b) __fmul_rn((a), (b))
#define FA(a, b) __fadd_rn((a), (b))
#define FS(a, b) __fsub_rn((a), (b))
#define FD(a, b) __fdiv_rn((a), (b))

// ----------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. 2011): key (seed_lo, seed_hi), counter
// (walk_lo, walk_hi, purpose, trial) (R2)
// ----------------------------------------------------------------------------
// MPG_ROLL_PHILOX: rolled rounds (the kernel inlines it at ~10 sites, ~500 SASS
// instructions unrolled): measured -2 % (configs[2]) / -3.5 % ([4]) walk time
#ifndef MPG_ROLL_PHILOX
#define MPG_ROLL_PHILOX 1
#endif
__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#if MPG_ROLL_PHILOX
#pragma unroll 1
#else
#pragma unroll
#endif
    for (int r = 0; r < 10; r++) {
        unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ uint4 rng_draw(uint64_t seed, uint64_t walk, uint32_t purpose, uint32_t trial) {
    return philox10(make_uint4((uint32_t)walk, (uint32_t)(walk >> 32), purpose, trial),
                    make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}
// (x>>8)*2^-24 and floor(x*m/2^32): both exact (R2)
__device__ __forceinline__ float u01(uint32_t x) { return (float)(x >> 8) * (1.0f / 16777216.0f); }
__device__ __forceinline__ uint32_t uidx(uint32_t x, uint32_t m) { return __umulhi(x, m); }

// ----------------------------------------------------------------------------
// scene records (passed by value as a kernel parameter)
// ----------------------------------------------------------------------------
#define DS_MAX_SURF 16
#define DS_MAX_LIGHT 8

struct DSurf {
    int kind, mat, tri_begin, tri_count;
    float eta_in, eta_out, refl, radius;
    float rough;   // GGX alpha of a glossy surface (0: pure specular, R37)
    float3 center, origin, eu, ev, nq; // nq: unit quad normal
};

struct DLight {
    int kind;
    float emit, pdf;            // pdf of x_L: 1/(area*n_light) (quad) or 1/n_light (point)
    float3 pos, eu, ev, n, l1, l2; // n: emission normal; l1,l2: orthonormal axes of the light plane
};

// Per-vertex arrays indexed by a rolled loop's counter.  With N <= MPG_SEL_MAX
// the access is a select chain over register-resident elements instead of a
// local-memory index; measured slower for k = 2 (configs[1] 67.6 -> 71.6 ms:
// more spills at the 80-register cap), so direct indexing is the default.
#ifndef MPG_SEL_MAX
#define MPG_SEL_MAX 0
#endif
template <typename T, int N> __device__ __forceinline__ T rget(const T (&a)[N], int i) {
    if constexpr (N <= MPG_SEL_MAX) {
        T r = a[0];
#pragma unroll
        for (int j = 1; j < N; j++)
            if (i == j) r = a[j];
        return r;
    } else {
        return a[i];
    }
}
template <typename T, int N> __device__ __forceinline__ void rset(T (&a)[N], int i, const T &v) {
    if constexpr (N <= MPG_SEL_MAX) {
#pragma unroll
        for (int j = 0; j < N; j++)
            if (i == j) a[j] = v;
    } else {
        a[i] = v;
    }
}
template <typename T, int N, int M> __device__ __forceinline__ T rget2(const T (&a)[N][M], int i, int c) {
    if constexpr (N <= MPG_SEL_MAX) {
        T r = a[0][c];
#pragma unroll
        for (int j = 1; j < N; j++)
            if (i == j) r = a[j][c];
        return r;
    } else {
        return a[i][c];
    }
}
template <typename T, int N, int M> __device__ __forceinline__ void rset2(T (&a)[N][M], int i, int c, T v) {
    if constexpr (N <= MPG_SEL_MAX) {
#pragma unroll
        for (int j = 0; j < N; j++)
            if (i == j) a[j][c] = v;
    } else {
        a[i][c] = v;
    }
}

// triangle record stride in float4: v0, v1, v2 (48 B; a 64-B record read with two
// 256-bit loads, LDG.E.ENL2.256, measured no faster on configs[1,2])
#define TSTRIDE 3

// BVH node layouts, chosen per scene at build time (DScene::bvh_w, template W of
// the traversal).  W = 2: binary SAH nodes, 4 float4 (64 B): two child boxes +
// two child refs.  W = 4: 4-wide nodes collapsed from the binary tree, 8 float4
// (128 B) SoA: lo_x[4], hi_x[4], lo_y[4], hi_y[4], lo_z[4], hi_z[4], child
// refs[4], pad; children sorted by entry distance.  Measured (k_walk ms, binary
// -> 4-wide): configs[1] (5 k tris) 41.8 -> 43.6, [2] (522 k) 322 -> 322,
// [3] (780 k) 283 -> 237, [4] 11.3 -> 11.1: half the dependent node fetches pay
// off once the tree is deep; the scene build picks 4-wide from 65,536 triangles
// (MPG_BVH_WIDTH=2|4 overrides).
// Child ref: >= 0 node index, < 0 leaf ~(first_tri << 3 | count - 1),
// 0x7fffffff empty slot (point box at 3e38: never entered).
#define NODE_F4(W) ((W) == 4 ? 8 : 4)
// load path of BVH nodes and leaf triangles in the traversal loop (experiment knob:
// __ldcg keeps them out of L1, leaving L1 to the lanes' local memory)
#ifndef MPG_LDN
#define MPG_LDN __ldg
#endif
#define TRAV_STACK(W) ((W) == 4 ? 96 : 64)
// MPG_TOP_NODES = N > 0: the walk kernel stages the first N nodes of the tree (the scene build numbers
// the top levels breadth-first, so these are the root's first levels) in shared memory and the
// traversal reads them there (north_star: "node stream staged through shared memory"; A/B in
// measured, not faster -- 0 = off)
#ifndef MPG_TOP_NODES
#define MPG_TOP_NODES 0
#endif

// One node visit of the ordered traversal: returns the nearest child whose box
// overlaps [tmin, tmax] (or pops the stack if none) and pushes the others
// far-to-near.  Same slab arithmetic for both layouts.
template <int W>
// Slab distances as one FFMA per plane: t = b * idir - oi with oi = o * idir
// precomputed per ray (Aila & Laine 2009).  The rounding of oi shifts a plane
// by ~ulp(|o|); node boxes are inflated by extent * 2^-20 at build time, so the
// test stays conservative (a box the ray truly enters is never culled).
__device__ __forceinline__ int bvh_visit(const float4 *nodes, int node, float3 oi, float3 idir, float tmin,
                                         float tmax, int *stack, int &sp, const float4 *top = nullptr) {
  if (W == 4) {
    const float4 *nd = nodes + NODE_F4(4) * node;
    float4 lx, hx, ly, hy, lz, hz;
    int4 ch;
    if (MPG_TOP_NODES > 0 && top && node < MPG_TOP_NODES) {   // the first levels, staged in shared memory
        const float4 *tn = top + NODE_F4(4) * node;
        lx = tn[0]; hx = tn[1]; ly = tn[2]; hy = tn[3]; lz = tn[4]; hz = tn[5];
        ch = *reinterpret_cast<const int4 *>(tn + 6);
    } else {
        lx = MPG_LDN(nd); hx = MPG_LDN(nd + 1); ly = MPG_LDN(nd + 2); hy = MPG_LDN(nd + 3); lz = MPG_LDN(nd + 4);
        hz = MPG_LDN(nd + 5);
        ch = MPG_LDN(reinterpret_cast<const int4 *>(nd + 6));
    }
    const float INF = __int_as_float(0x7f800000);
    float t[4];
    int c[4] = {ch.x, ch.y, ch.z, ch.w};
#define MPG_SLAB(J, LX, HX, LY, HY, LZ, HZ)                                                         \
    {                                                                                                \
        float x0 = fmaf(LX, idir.x, -oi.x), x1 = fmaf(HX, idir.x, -oi.x);                            \
        float y0 = fmaf(LY, idir.y, -oi.y), y1 = fmaf(HY, idir.y, -oi.y);                            \
        float z0 = fmaf(LZ, idir.z, -oi.z), z1 = fmaf(HZ, idir.z, -oi.z);                            \
        float tn = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), tmin));           \
        float tf = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), tmax));           \
        t[J] = tn <= tf ? tn : INF;                                                                  \
    }
    MPG_SLAB(0, lx.x, hx.x, ly.x, hy.x, lz.x, hz.x)
    MPG_SLAB(1, lx.y, hx.y, ly.y, hy.y, lz.y, hz.y)
    MPG_SLAB(2, lx.z, hx.z, ly.z, hy.z, lz.z, hz.z)
    MPG_SLAB(3, lx.w, hx.w, ly.w, hy.w, lz.w, hz.w)
#undef MPG_SLAB
#define MPG_CAS(A, B)                                                                                \
    {                                                                                                \
        bool sw = t[B] < t[A];                                                                       \
        float ta = sw ? t[B] : t[A], tb = sw ? t[A] : t[B];                                          \
        int ca = sw ? c[B] : c[A], cb = sw ? c[A] : c[B];                                            \
        t[A] = ta; t[B] = tb; c[A] = ca; c[B] = cb;                                                  \
    }
    MPG_CAS(0, 1) MPG_CAS(2, 3) MPG_CAS(0, 2) MPG_CAS(1, 3) MPG_CAS(1, 2)
#undef MPG_CAS
    MPG_CHECK(sp >= 1 && sp + 3 <= TRAV_STACK(4));
    if (t[0] == INF) return stack[--sp];
    if (t[3] != INF) stack[sp++] = c[3];
    if (t[2] != INF) stack[sp++] = c[2];
    if (t[1] != INF) stack[sp++] = c[1];
    return c[0];
  } else {
    const float4 *nd = nodes + NODE_F4(2) * node;
    float4 a, b, c;
    int4 ch;
    if (MPG_TOP_NODES > 0 && top && node < MPG_TOP_NODES) {
        const float4 *tn = top + NODE_F4(2) * node;
        a = tn[0]; b = tn[1]; c = tn[2];
        ch = *reinterpret_cast<const int4 *>(tn + 3);
    } else {
        a = MPG_LDN(nd); b = MPG_LDN(nd + 1); c = MPG_LDN(nd + 2);
        ch = MPG_LDN(reinterpret_cast<const int4 *>(nd + 3));
    }
    float tx0 = fmaf(a.x, idir.x, -oi.x), tx1 = fmaf(a.w, idir.x, -oi.x);
    float ty0 = fmaf(a.y, idir.y, -oi.y), ty1 = fmaf(b.x, idir.y, -oi.y);
    float tz0 = fmaf(a.z, idir.z, -oi.z), tz1 = fmaf(b.y, idir.z, -oi.z);
    float n0 = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), tmin));
    float f0 = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tmax));
    float sx0 = fmaf(b.z, idir.x, -oi.x), sx1 = fmaf(c.y, idir.x, -oi.x);
    float sy0 = fmaf(b.w, idir.y, -oi.y), sy1 = fmaf(c.z, idir.y, -oi.y);
    float sz0 = fmaf(c.x, idir.z, -oi.z), sz1 = fmaf(c.w, idir.z, -oi.z);
    float n1 = fmaxf(fmaxf(fminf(sx0, sx1), fminf(sy0, sy1)), fmaxf(fminf(sz0, sz1), tmin));
    float f1 = fminf(fminf(fmaxf(sx0, sx1), fmaxf(sy0, sy1)), fminf(fmaxf(sz0, sz1), tmax));
    bool h0 = n0 <= f0, h1 = n1 <= f1;
    MPG_CHECK(sp >= 1 && sp + 1 <= TRAV_STACK(2));
    if (h0 && h1) {
        bool swp = n1 < n0;
        stack[sp++] = swp ? ch.x : ch.y;
        return swp ? ch.y : ch.x;
    }
    if (h0) return ch.x;
    if (h1) return ch.y;
    return stack[--sp];
  }
}

struct DScene {
    int n_surf, n_light, n_tri, n_nodes;
    int bvh_w;           // 2 or 4: node layout (see bvh_visit)
    float extent;
    DSurf surf[DS_MAX_SURF];
    DLight light[DS_MAX_LIGHT];
    const float4 *nodes; // NODE_F4(bvh_w) float4 per node (see bvh_visit)
    const float4 *tpos;  // BVH order, TSTRIDE float4 per tri; v0.w = original tri id, v1.w = surf id, v2.w = specular flag
    const float4 *tnrm;  // BVH order, 3 float4 per tri: vertex shading normals
    const int4 *oidx;    // original order: vertex indices (w: BVH slot)
    const int4 *tadj;    // BVH order: BVH slots of the neighbours across the edges opposite v0, v1, v2 (-1: none)
    const float4 *vpos;  // original vertex positions
};

// A hit / chain vertex: prim = BVH-order triangle slot (>= 0) or -1 (analytic)
struct Hit {
    float t;
    int prim, surf;
    float3 p;
};

// per-lane work counters (reduced once per kernel)
struct LaneStats {
    uint32_t rays, nodes, tris;
};

// ----------------------------------------------------------------------------
// intersection
// ----------------------------------------------------------------------------
struct RayW {
    float3 o, d, idir;
    int kx, ky, kz;
    float Sx, Sy, Sz;
};

__device__ __forceinline__ void ray_setup(RayW &r, float3 o, float3 d) {
    r.o = o;
    r.d = d;
    r.idir = f3(d.x != 0.0f ? 1.0f / d.x : copysignf(1e30f, d.x), d.y != 0.0f ? 1.0f / d.y : copysignf(1e30f, d.y),
                d.z != 0.0f ? 1.0f / d.z : copysignf(1e30f, d.z));
    float ax = fabsf(d.x), ay = fabsf(d.y), az = fabsf(d.z);
    int kz = (ax > ay) ? (ax > az ? 0 : 2) : (ay > az ? 1 : 2);
    int kx = kz == 2 ? 0 : kz + 1;
    int ky = kx == 2 ? 0 : kx + 1;
    if (comp(d, kz) < 0.0f) { int t = kx; kx = ky; ky = t; }
    r.kx = kx; r.ky = ky; r.kz = kz;
    float dz = comp(d, kz);
    r.Sx = comp(d, kx) / dz;
    r.Sy = comp(d, ky) / dz;
    r.Sz = 1.0f / dz;
}

// Watertight ray/triangle test (Woop, Benthin, Wald 2013), double-sided.  The
// edge functions use non-contracted products so a shared edge evaluates to
// exactly opposite values in both triangles (no cracks for reprojection rays).
__device__ __forceinline__ bool tri_hit(const RayW &r, float3 v0, float3 v1, float3 v2, float tmin, float tmax,
                                        float &t, float &b0, float &b1, float &b2) {
    float3 A = v0 - r.o, B = v1 - r.o, C = v2 - r.o;
    float Akz = comp(A, r.kz), Bkz = comp(B, r.kz), Ckz = comp(C, r.kz);
    float Ax = comp(A, r.kx) - r.Sx * Akz, Ay = comp(A, r.ky) - r.Sy * Akz;
    float Bx = comp(B, r.kx) - r.Sx * Bkz, By = comp(B, r.ky) - r.Sy * Bkz;
    float Cx = comp(C, r.kx) - r.Sx * Ckz, Cy = comp(C, r.ky) - r.Sy * Ckz;
    float U = __fsub_rn(__fmul_rn(Cx, By), __fmul_rn(Cy, Bx));
    float V = __fsub_rn(__fmul_rn(Ax, Cy), __fmul_rn(Ay, Cx));
    float W = __fsub_rn(__fmul_rn(Bx, Ay), __fmul_rn(By, Ax));
    if ((U < 0.0f || V < 0.0f || W < 0.0f) && (U > 0.0f || V > 0.0f || W > 0.0f)) return false;
    float det = U + V + W;
    if (det == 0.0f) return false;
    float T = U * (r.Sz * Akz) + V * (r.Sz * Bkz) + W * (r.Sz * Ckz);
    float inv = 1.0f / det;
    t = T * inv;
    if (!(t > tmin && t < tmax)) return false;
    b0 = U * inv; b1 = V * inv; b2 = W * inv;
    return true;
}

// Ray/sphere in fp64 (a few DP flops per analytic surface): the reprojected
// vertex must be accurate to ~1 ulp of its fp32 coordinates, because near
// grazing reflection the residual's sensitivity to position is ~1/(2cos theta)
// larger than nominal and o + t*d in fp32 stalls Newton at ||C|| ~ 2e-5 (measured).
__device__ __forceinline__ bool sphere_hit(float3 o, float3 d, float3 c, float R, float tmin, float tmax, float &t,
                                           float3 &p) {
    double ox = (double)o.x - c.x, oy = (double)o.y - c.y, oz = (double)o.z - c.z;
    double dx = d.x, dy = d.y, dz = d.z;
    double dd = dx * dx + dy * dy + dz * dz;
    double b = (ox * dx + oy * dy + oz * dz) / dd;
    double qx = ox - b * dx, qy = oy - b * dy, qz = oz - b * dz;
    double disc = ((double)R * R - (qx * qx + qy * qy + qz * qz)) / dd;
    if (disc < 0.0) return false;
    double sq = sqrt(disc);
    double t0 = -b - sq, t1 = -b + sq, tt;
    if (t0 > tmin && t0 < tmax) tt = t0;
    else if (t1 > tmin && t1 < tmax) tt = t1;
    else return false;
    t = (float)tt;
    p = make_float3((float)((double)o.x + tt * dx), (float)((double)o.y + tt * dy), (float)((double)o.z + tt * dz));
    return true;
}

__device__ __forceinline__ bool quad_hit(float3 o, float3 d, float3 q0, float3 e1, float3 e2, float tmin, float tmax,
                                         float &t) {
    float3 pv = cross(d, e2);
    float det = dot(e1, pv);
    if (det == 0.0f) return false;
    float inv = 1.0f / det;
    float3 tv = o - q0;
    float u = dot(tv, pv) * inv;
    if (u < 0.0f || u > 1.0f) return false;
    float3 qv = cross(tv, e1);
    float v = dot(d, qv) * inv;
    if (v < 0.0f || v > 1.0f) return false;
    float tt = dot(e2, qv) * inv;
    if (!(tt > tmin && tt < tmax)) return false;
    t = tt;
    return true;
}

// Closest hit (ANY false) or any hit (ANY true) with t in (tmin, tmax) over all
// surfaces, or only specular ones (spec_only): the operator r(x, w) of Eq. 6
// and the visibility V of Eq. 2.
#if defined(MPG_TIMELINE) && !defined(MPG_NH)
#define MPG_NH
#endif
#ifdef MPG_NH
__device__ unsigned long long g_nh[256];   // diagnostic: closest-hit rays by node visits
#endif
// WANT_P = false: for a triangle hit h.p holds the hit's barycentrics instead of the fp32 point
// (the walk recomputes the point in fp64 from the vertices anyway, refine_hit: three 16-byte
// loads per ray less on the L1 data pipe, the unit that bounds the traversal)
template <int W, bool WANT_P = true>
__device__ __forceinline__ bool trace(const DScene &S, float3 o, float3 d, float tmin, float tmax, bool spec_only,
                                      const bool ANY, Hit &h, LaneStats &st, int hint = -1,
                                      const float4 *top = nullptr) {   // callers count rays
#ifdef MPG_NH
    const uint32_t n_at_entry = st.nodes;
#endif
    float best = tmax;
    int bprim = -2, bsurf = -1;
    float bb0 = 0.f, bb1 = 0.f, bb2 = 0.f;
    float3 bp = f3(0.f, 0.f, 0.f);
    for (int i = 0; i < S.n_surf; i++) {
        const DSurf &f = S.surf[i];
        if (f.kind == 2 || (spec_only && f.mat == 2)) continue;
        float t;
        float3 p;
        bool hit;
        if (f.kind == 0) hit = sphere_hit(o, d, f.center, f.radius, tmin, best, t, p);
        else {
            hit = quad_hit(o, d, f.origin, f.eu, f.ev, tmin, best, t);
            p = o + d * t;
        }
        if (hit) {
            best = t; bprim = -1; bsurf = i; bp = p;
            if (ANY) { h.t = t; h.prim = -1; h.surf = i; return true; }
        }
    }
    if (S.n_tri > 0) {
        // while-while traversal with postponed leaves (Aila & Laine 2009): lanes
        // keep visiting inner nodes together until every active lane has a leaf
        // waiting, then intersect leaves together -- node visits and triangle
        // tests execute with most lanes of the warp active.
        const int SENT = 0x7fffffff, NONE = 0;
        RayW r;
        ray_setup(r, o, d);
        if (!ANY && hint >= 0) {
            // Bound the search by the hit on a hinted triangle (the chain vertex's current
            // triangle on a reprojection ray): the traversal below then only enters boxes
            // closer than that hit.  The closest hit is unchanged (strict t < best), except
            // that among hits at exactly equal t the hinted one is kept (shared edges, R17).
            st.tris++;
            float4 p0 = __ldg(S.tpos + TSTRIDE * hint), p1 = __ldg(S.tpos + TSTRIDE * hint + 1),
                   p2 = __ldg(S.tpos + TSTRIDE * hint + 2);
            float t, c0, c1, c2;
            if (!(spec_only && __float_as_int(p2.w) == 0) &&
                tri_hit(r, xyz(p0), xyz(p1), xyz(p2), tmin, best, t, c0, c1, c2)) {
                best = t; bprim = hint; bsurf = __float_as_int(p1.w);
                bb0 = c0; bb1 = c1; bb2 = c2;
            }
        }
        const float3 oi = f3(o.x * r.idir.x, o.y * r.idir.y, o.z * r.idir.z);
        int stack[TRAV_STACK(W)];
        stack[0] = SENT;
        int sp = 1;
        int node = 0, leaf = NONE;
        while (node != SENT || leaf != NONE) {
            while (node >= 0 && node != SENT) {
                st.nodes++;
                MPG_CHECK(node < S.n_nodes);
                node = bvh_visit<W>(S.nodes, node, oi, r.idir, tmin, best, stack, sp, top);
                if (node < 0 && leaf == NONE) { // postpone the leaf, keep traversing
                    leaf = node;
                    node = stack[--sp];
                }
                if (!__any_sync(__activemask(), leaf == NONE)) break;
            }
            while (leaf != NONE) {
                int v = ~leaf;
                int start = v >> 3, cnt = (v & 7) + 1;
                MPG_CHECK(start >= 0 && start + cnt <= S.n_tri);
                for (int j = start; j < start + cnt; j++) {
                    st.tris++;
                    float4 p0 = MPG_LDN(S.tpos + TSTRIDE * j), p1 = MPG_LDN(S.tpos + TSTRIDE * j + 1),
                           p2 = MPG_LDN(S.tpos + TSTRIDE * j + 2);
                    if (spec_only && __float_as_int(p2.w) == 0) continue;
                    float t, c0, c1, c2;
                    if (tri_hit(r, xyz(p0), xyz(p1), xyz(p2), tmin, best, t, c0, c1, c2)) {
                        best = t; bprim = j; bsurf = __float_as_int(p1.w);
                        bb0 = c0; bb1 = c1; bb2 = c2;
                        if (ANY) { h.t = t; h.prim = j; h.surf = bsurf; return true; }
                    }
                }
                leaf = NONE;
                if (node < 0) { // the traversal stopped on another leaf
                    leaf = node;
                    node = stack[--sp];
                }
            }
        }
    }
    if (ANY) return false;
#ifdef MPG_NH
    atomicAdd(&g_nh[min(st.nodes - n_at_entry, 255u)], 1ull);
#endif
    h.t = best; h.prim = bprim; h.surf = bsurf;
    if (bsurf < 0) return false;
    if (bprim >= 0) {
        if constexpr (WANT_P) {
            // hit point from barycentrics: lies on the triangle plane up to rounding
            float3 v0 = xyz(__ldg(S.tpos + TSTRIDE * bprim)), v1 = xyz(__ldg(S.tpos + TSTRIDE * bprim + 1)),
                   v2 = xyz(__ldg(S.tpos + TSTRIDE * bprim + 2));
            h.p = v0 * bb0 + v1 * bb1 + v2 * bb2;
        } else {
            h.p = f3(bb0, bb1, bb2);
        }
    } else {
        h.p = bp;
    }
    return true;
}

// ----------------------------------------------------------------------------
// local geometry at a chain vertex (R3, R4, R9)
// ----------------------------------------------------------------------------
__device__ __forceinline__ float3 geo_normal(const DScene &S, int prim, int surf, float3 p) {
    const DSurf &f = S.surf[surf];
    if (prim >= 0) {
        float3 v0 = xyz(__ldg(S.tpos + TSTRIDE * prim)), v1 = xyz(__ldg(S.tpos + TSTRIDE * prim + 1)),
               v2 = xyz(__ldg(S.tpos + TSTRIDE * prim + 2));
        return nrmz(cross(v1 - v0, v2 - v0));
    }
    if (f.kind == 0) return nrmz(p - f.center);
    return f.nq;
}

// shading normal n_s and its derivatives along two tangent vectors a, b.
// mesh: Phong n = n~/|n~|, n~ = sum b_j n_j (BASELINE configs[1]); sphere: (p-c)/|p-c|.
__device__ __forceinline__ float3 shading(const DScene &S, int prim, int surf, float3 p, float3 a, float3 b,
                                          float3 &dna, float3 &dnb) {
    if (prim >= 0) {
        float3 v0 = xyz(__ldg(S.tpos + TSTRIDE * prim)), v1 = xyz(__ldg(S.tpos + TSTRIDE * prim + 1)),
               v2 = xyz(__ldg(S.tpos + TSTRIDE * prim + 2));
        float3 n0 = xyz(__ldg(S.tnrm + 3 * prim)), n1 = xyz(__ldg(S.tnrm + 3 * prim + 1)),
               n2 = xyz(__ldg(S.tnrm + 3 * prim + 2));
        float3 e1 = v1 - v0, e2 = v2 - v0;
        float3 Ng = cross(e1, e2);
        float inv = 1.0f / dot(Ng, Ng);
        float3 g1 = cross(e2, Ng) * inv, g2 = cross(Ng, e1) * inv; // barycentric gradients
        float3 r = p - v0;
        float c1 = dot(r, g1), c2 = dot(r, g2), c0 = 1.0f - c1 - c2;
        float3 nt = n0 * c0 + n1 * c1 + n2 * c2;
        float il = rsqrtf(dot(nt, nt));
        float3 n = nt * il;
        float3 d1 = n1 - n0, d2 = n2 - n0;
        float3 ta = d1 * dot(a, g1) + d2 * dot(a, g2);
        float3 tb = d1 * dot(b, g1) + d2 * dot(b, g2);
        dna = (ta - n * dot(n, ta)) * il;
        dnb = (tb - n * dot(n, tb)) * il;
        return n;
    }
    const DSurf &f = S.surf[surf];
    if (f.kind == 0) {
        float3 r = p - f.center;
        float il = rsqrtf(dot(r, r));
        float3 n = r * il;
        dna = (a - n * dot(n, a)) * il;
        dnb = (b - n * dot(n, b)) * il;
        return n;
    }
    dna = f3(0.f, 0.f, 0.f);
    dnb = dna;
    return f.nq;
}

__device__ __forceinline__ float3 shading_normal(const DScene &S, int prim, int surf, float3 p) {
    float3 da, db;
    return shading(S, prim, surf, p, f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 0.f), da, db);
}

// unpolarized dielectric Fresnel reflectance (eta1 = medium of incidence)
__device__ __forceinline__ float fresnel(float ci, float eta1, float eta2) {
    ci = fabsf(ci);
    float e = eta1 / eta2;
    float st2 = e * e * (1.0f - ci * ci);
    if (st2 >= 1.0f) return 1.0f;
    float ct = sqrtf(1.0f - st2);
    float rs = (eta1 * ci - eta2 * ct) / (eta1 * ci + eta2 * ct);
    float rp = (eta2 * ci - eta1 * ct) / (eta2 * ci + eta1 * ct);
    return 0.5f * (rs * rs + rp * rp);
}
