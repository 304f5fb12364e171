/*
 * mpg_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU oracle of the batched manifold walk of
 * Fan et al., "Manifold Path Guiding for Importance Sampling Specular Chains"
 * (arXiv 2311.12818).  It computes in fp64 (reading R24) except the seed
 * arithmetic, which is fp32 without contraction (reading R23), and follows the
 * algorithm step by step in the paper's order:
 *   light sample x_L            PAPER.md:337  (§5.1 "x_L by uniformly sampling all emitters")
 *   seed chain sampling         PAPER.md:395-421 (§5.4 init, Eq. 8), :501-512 (Eq. 13, alpha=0.5)
 *   deduction recursion         PAPER.md:374-380 (Eq. 6)
 *   manifold walk               PAPER.md:240-243 (Newton + reprojection), :362 (quadratic conv.)
 *   throughput T = kappa G L    PAPER.md:229-237 (Eq. 2)
 *   reciprocal probability      PAPER.md:582-591 (Eq. 15, trials reuse n)
 *   sample weight w = T <1/P>   PAPER.md:427-432 (Eq. 9), estimator Eq. 3 (:267-277)
 *   guide tables                PAPER.md:434-466 (Eqs. 10-11) as the BASELINE.json histogram
 *   STree + vMF guide           PAPER.md:424-530 (Eqs. 9-12, STree P:518-523)      [R28-R31]
 *   repeated reciprocal est.    PAPER.md:906-915 (R x M)                            [R32]
 *   photon-based p_0            PAPER.md:398, :883                                   [R33]
 *   glossy separator weighting  PAPER.md:550-556 (Eq. 14)                            [R35]
 *   selective activation        PAPER.md:604-608                                     [R36]
 *   glossy chains (offsets)     PAPER.md:562-565                                     [R37]
 * Every choice the paper leaves open is a numbered reading (R1..R35) in
 * DESIGN.md §3; the code cites them as [Rn].
 *
 * It shares no code, header, table or constant generator with the CUDA
 * library under paper_2311_12818_b200/csrc; neither includes the other.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may load it.
 *
 * Library primitives used as steps: dense LU with partial pivoting (the plain
 * definition of "solve J d = -C"), a median-split BVH (an acceleration
 * structure whose closest hit equals brute force; pinned in tests).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KMAX 8
#define ST_CONVERGED 0
#define ST_MAXITER 1
#define ST_SEED_FAIL 2
#define ST_BAD_SIDE 3
#define ST_DEGENERATE 4
#define ST_OCCLUDED 5
#define ST_INACTIVE 6 /* selective activation: no own sample in the STree leaf [R36] */

/* ------------------------------------------------------------------------ */
/* input records (mirrored by oracle/oracle.py ctypes)                       */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t kind, mat, tri_begin, tri_count; /* kind 0 sphere 1 quad 2 mesh; mat 0 conductor 1 dielectric 2 diffuse */
    float eta_in, eta_out, reflectance, radius;
    float center[3], origin[3], edge_u[3], edge_v[3];
    float roughness; /* GGX alpha of a glossy specular surface (0: pure specular) [R37] */
} orc_surface;

typedef struct {
    int32_t kind; /* 0 point, 1 quad area (one-sided along edge_u x edge_v) */
    float emit;
    float position[3], edge_u[3], edge_v[3];
} orc_light;

typedef struct {
    int32_t mode;     /* 0 cap, 1 triangle, 2 guide-uv */
    int32_t surf_id;
    int32_t k;
    uint32_t tau;     /* bit i = 1 <=> vertex i+1 is T */
    float grid_origin[2], grid_extent[2];
    int32_t cells_x, cells_y, bins_x, bins_y;
    float uv_origin[2], uv_scale[2], uv_plane_y;
    const uint64_t *prefix; /* [cells][bins] inclusive prefix sums of W' (orc_guide_tables) */
    /* mode 3 (typed direction guide, configs[4]; orc_guide_dir_tables) */
    const uint64_t *n_prefix;    /* [cells][6] defensive length mixture (Eqs. 10, 13)  */
    const uint64_t *type_prefix; /* [cells][126] per-length type weights (Eq. 11)      */
    const uint32_t *dir_prefix;  /* [cells][126][bins] learned direction weights        */
    /* mode 4 (STree + vMF guide; orc_stree_build): n_prefix / type_prefix
       above are then per leaf; the tree is descended with (x_D, x_L) */
    int32_t root_ref, pad_;      /* >= 0 inner node, < 0: ~leaf                          */
    const void *nodes;           /* orc_snode [n_nodes]                                  */
    const int32_t *grp_off;      /* [leaves][127] lobe offsets of the (leaf, type) groups */
    const uint64_t *lobe_prefix; /* [lobes] inclusive per-group prefix of lobe weights   */
    const float *lobe_mu;        /* [lobes][4] vMF mean direction (xyz), kappa (w)       */
    const int64_t *leaf_own;     /* [leaves] samples whose own key lies in the leaf (no copies) */
} orc_seed_cfg;

typedef struct {
    int32_t max_iters;
    int32_t trials;
    uint32_t k_max;
    int32_t max_iters_long; /* cap for chains with k >= 3 (0: max_iters) */
    double tol, beta0, same_chain_eps, ray_eps;
    uint64_t seed, walk_id_base;
    int32_t recip_repeats;  /* M >= 2: M independent reciprocal estimates averaged [R32] */
    int32_t selective;      /* selective activation [R36]: with the STree guide, a walk whose
                               leaf holds no own (non-copy) sample is INACTIVE (left to path tracing) */
} orc_opts;

typedef struct {
    int32_t status, iters;
    uint32_t trials;
    int32_t truncated;
    double G, T, kappa, w;
    double pos[KMAX][3];
    int32_t prim[KMAX], surf[KMAX];
    double xL[3];
    double pdfL;
    float target[3];
    int32_t bin;
    int64_t total_iters; /* Newton iterations over the primary and all trials */
    int64_t attempts;    /* seed draws (primary + trials) */
    int32_t k;           /* chain length n of the primary */
    uint32_t tau;        /* resolved type string of the primary (bit i: vertex i+1 is T) */
    double Pn;           /* P(n) of the defensive length mixture (1 for fixed-length configs) */
} orc_walk_out;

/* ------------------------------------------------------------------------ */
/* fp64 vectors                                                               */
/* ------------------------------------------------------------------------ */
typedef struct { double x, y, z; } v3;
static v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 vf(const float *f) { return V(f[0], f[1], f[2]); }
static v3 add(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 mul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 cross(v3 a, v3 b) { return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
static double len(v3 a) { return sqrt(dot(a, a)); }
static v3 nrmz(v3 a) { return mul(a, 1.0 / len(a)); }
static double vget(v3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

/* Orthonormal basis of a unit vector (Duff et al. 2017, "Building an
 * Orthonormal Basis, Revisited") -- any basis is valid [R3,R4]. */
static void onb(v3 n, v3 *b1, v3 *b2) {
    double sign = copysign(1.0, n.z);
    double a = -1.0 / (sign + n.z);
    double b = n.x * n.y * a;
    *b1 = V(1.0 + sign * n.x * n.x * a, sign * b, -sign * n.x);
    *b2 = V(b, sign + n.y * n.y * a, -n.y);
}

/* the derivative of that basis for a change dn of n (differentiating the formulas above);
 * glossy vertices need it: with an offset normal the frame's twist no longer drops out of
 * the constraint at the solution [R37] */
static void onb_d(v3 n, v3 dn, v3 *d1, v3 *d2) {
    double sign = copysign(1.0, n.z);
    double a = -1.0 / (sign + n.z);
    double da = a * a * dn.z;
    double db = (dn.x * n.y + n.x * dn.y) * a + n.x * n.y * da;
    *d1 = V(sign * (2.0 * n.x * dn.x * a + n.x * n.x * da), sign * db, -sign * dn.x);
    *d2 = V(db, 2.0 * n.y * dn.y * a + n.y * n.y * da, -dn.y);
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al. 2011), key=(seed_lo,seed_hi),                 */
/* counter=(walk_lo, walk_hi, purpose, trial)  [R2]                           */
/* ------------------------------------------------------------------------ */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (r < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void orc_philox_batch(const uint32_t *ctr, int64_t n, const uint32_t key[2], uint32_t *out) {
    for (int64_t i = 0; i < n; i++) orc_philox(ctr + 4 * i, key, out + 4 * i);
}

static void draw(const orc_opts *o, uint64_t walk, uint32_t purpose, uint32_t trial, uint32_t out[4]) {
    uint32_t ctr[4] = {(uint32_t)walk, (uint32_t)(walk >> 32), purpose, trial};
    uint32_t key[2] = {(uint32_t)o->seed, (uint32_t)(o->seed >> 32)};
    orc_philox(ctr, key, out);
}

/* u32 -> [0,1): (x>>8)*2^-24, exact [R2] */
static float u01(uint32_t x) { return (float)(x >> 8) * (1.0f / 16777216.0f); }
/* index in [0,m): floor(x*m/2^32), exact [R2] */
static uint32_t uidx(uint32_t x, uint32_t m) { return (uint32_t)(((uint64_t)x * m) >> 32); }

/* ------------------------------------------------------------------------ */
/* scene                                                                      */
/* ------------------------------------------------------------------------ */
typedef struct { double lo[3], hi[3]; int32_t left, right, first, count; } bnode;

typedef struct {
    int n_surf, n_vert, n_tri, n_light;
    orc_surface *surf;
    orc_light *light;
    double *P, *N; /* [n_vert*3] */
    int32_t *I;    /* [n_tri*3] */
    int32_t *TS;   /* [n_tri] */
    int32_t *order;
    bnode *nodes;
    int n_nodes;
    double extent;
} orc_scene;

static v3 vtx(const orc_scene *s, int i) { return V(s->P[3 * i], s->P[3 * i + 1], s->P[3 * i + 2]); }
static v3 vnr(const orc_scene *s, int i) { return V(s->N[3 * i], s->N[3 * i + 1], s->N[3 * i + 2]); }

static const double *g_cent; static int g_axis;
static int cmp_cent(const void *a, const void *b) {
    double ca = g_cent[3 * (*(const int32_t *)a) + g_axis], cb = g_cent[3 * (*(const int32_t *)b) + g_axis];
    if (ca < cb) return -1;
    if (ca > cb) return 1;
    return (*(const int32_t *)a) - (*(const int32_t *)b);
}

static int build_node(orc_scene *s, const double *cent, int first, int count) {
    int id = s->n_nodes++;
    bnode *nd = &s->nodes[id];
    for (int a = 0; a < 3; a++) { nd->lo[a] = 1e300; nd->hi[a] = -1e300; }
    double clo[3] = {1e300, 1e300, 1e300}, chi[3] = {-1e300, -1e300, -1e300};
    for (int j = first; j < first + count; j++) {
        int t = s->order[j];
        for (int c = 0; c < 3; c++) {
            int vi = s->I[3 * t + c];
            for (int a = 0; a < 3; a++) {
                double v = s->P[3 * vi + a];
                if (v < nd->lo[a]) nd->lo[a] = v;
                if (v > nd->hi[a]) nd->hi[a] = v;
            }
        }
        for (int a = 0; a < 3; a++) {
            if (cent[3 * t + a] < clo[a]) clo[a] = cent[3 * t + a];
            if (cent[3 * t + a] > chi[a]) chi[a] = cent[3 * t + a];
        }
    }
    if (count <= 4) { nd->left = nd->right = -1; nd->first = first; nd->count = count; return id; }
    int axis = 0;
    for (int a = 1; a < 3; a++) if (chi[a] - clo[a] > chi[axis] - clo[axis]) axis = a;
    g_cent = cent; g_axis = axis;
    qsort(s->order + first, (size_t)count, sizeof(int32_t), cmp_cent); /* median split */
    int half = count / 2;
    int l = build_node(s, cent, first, half);
    int r = build_node(s, cent, first + half, count - half);
    nd = &s->nodes[id];
    nd->left = l; nd->right = r; nd->first = first; nd->count = 0;
    return id;
}

void orc_scene_destroy(void *h) {
    orc_scene *s = (orc_scene *)h;
    if (!s) return;
    free(s->surf); free(s->light); free(s->P); free(s->N); free(s->I); free(s->TS); free(s->order); free(s->nodes);
    free(s);
}

/* Copies everything; builds a median-split BVH over all mesh triangles. */
void *orc_scene_create(const orc_surface *surf, int n_surf, const float *pos, const float *nrm, int n_vert,
                       const int32_t *idx, const int32_t *tri_surf, int n_tri, const orc_light *light, int n_light) {
    orc_scene *s = (orc_scene *)calloc(1, sizeof(orc_scene));
    s->n_surf = n_surf; s->n_vert = n_vert; s->n_tri = n_tri; s->n_light = n_light;
    s->surf = (orc_surface *)malloc(sizeof(orc_surface) * (size_t)(n_surf > 0 ? n_surf : 1));
    memcpy(s->surf, surf, sizeof(orc_surface) * (size_t)n_surf);
    s->light = (orc_light *)malloc(sizeof(orc_light) * (size_t)(n_light > 0 ? n_light : 1));
    memcpy(s->light, light, sizeof(orc_light) * (size_t)n_light);
    s->P = (double *)malloc(sizeof(double) * 3 * (size_t)(n_vert + 1));
    s->N = (double *)malloc(sizeof(double) * 3 * (size_t)(n_vert + 1));
    for (int i = 0; i < 3 * n_vert; i++) { s->P[i] = pos[i]; s->N[i] = nrm[i]; }
    s->I = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)(n_tri + 1));
    s->TS = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_tri + 1));
    memcpy(s->I, idx, sizeof(int32_t) * 3 * (size_t)n_tri);
    memcpy(s->TS, tri_surf, sizeof(int32_t) * (size_t)n_tri);
    s->order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_tri + 1));
    s->nodes = (bnode *)malloc(sizeof(bnode) * (size_t)(2 * n_tri + 2));
    s->n_nodes = 0;
    if (n_tri > 0) {
        double *cent = (double *)malloc(sizeof(double) * 3 * (size_t)n_tri);
        for (int t = 0; t < n_tri; t++) {
            s->order[t] = t;
            for (int a = 0; a < 3; a++)
                cent[3 * t + a] = (s->P[3 * s->I[3 * t] + a] + s->P[3 * s->I[3 * t + 1] + a] + s->P[3 * s->I[3 * t + 2] + a]) / 3.0;
        }
        build_node(s, cent, 0, n_tri);
        free(cent);
    }
    /* scene extent: bbox diagonal of all surfaces and lights [R10] */
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
#define GROW(p) do { for (int a_ = 0; a_ < 3; a_++) { double q_ = vget((p), a_); if (q_ < lo[a_]) lo[a_] = q_; if (q_ > hi[a_]) hi[a_] = q_; } } while (0)
    for (int i = 0; i < n_surf; i++) {
        const orc_surface *f = &surf[i];
        if (f->kind == 0) { v3 c = vf(f->center); GROW(sub(c, V(f->radius, f->radius, f->radius))); GROW(add(c, V(f->radius, f->radius, f->radius))); }
        else if (f->kind == 1) { v3 o = vf(f->origin), u = vf(f->edge_u), w = vf(f->edge_v); GROW(o); GROW(add(o, u)); GROW(add(o, w)); GROW(add(add(o, u), w)); }
        else for (int t = f->tri_begin; t < f->tri_begin + f->tri_count; t++) for (int c = 0; c < 3; c++) GROW(vtx(s, s->I[3 * t + c]));
    }
    for (int i = 0; i < n_light; i++) {
        const orc_light *l = &light[i];
        v3 c = vf(l->position);
        if (l->kind == 1) {
            v3 u = mul(vf(l->edge_u), 0.5), w = mul(vf(l->edge_v), 0.5);
            GROW(add(add(c, u), w)); GROW(sub(sub(c, u), w)); GROW(add(sub(c, u), w)); GROW(sub(add(c, u), w));
        } else GROW(c);
    }
#undef GROW
    s->extent = len(sub(V(hi[0], hi[1], hi[2]), V(lo[0], lo[1], lo[2])));
    return s;
}

double orc_scene_extent(const void *h) { return ((const orc_scene *)h)->extent; }

/* ------------------------------------------------------------------------ */
/* ray intersection: r(x, w) of Eq. 6 and V of Eq. 2          */
/* ------------------------------------------------------------------------ */
typedef struct { double t; int prim, surf; v3 p; } hit_t;

/* Moller-Trumbore, double-sided; returns t or -1; u,v barycentric */
static double tri_isect(v3 o, v3 d, v3 v0, v3 e1, v3 e2, double *pu, double *pv, int quad) {
    v3 pvec = cross(d, e2);
    double det = dot(e1, pvec);
    if (det == 0.0) return -1.0;
    double inv = 1.0 / det;
    v3 tvec = sub(o, v0);
    double u = dot(tvec, pvec) * inv;
    if (u < 0.0 || u > 1.0) return -1.0;
    v3 qvec = cross(tvec, e1);
    double v = dot(d, qvec) * inv;
    if (v < 0.0 || (quad ? v > 1.0 : u + v > 1.0)) return -1.0;
    if (pu) *pu = u;
    if (pv) *pv = v;
    return dot(e2, qvec) * inv;
}

static int surf_is_specular(const orc_scene *s, int sid) { return s->surf[sid].mat != 2; }

/* analytic surfaces, brute force; updates best if closer */
static void isect_analytic(const orc_scene *s, v3 o, v3 d, double tmin, int spec_only, hit_t *best) {
    for (int i = 0; i < s->n_surf; i++) {
        const orc_surface *f = &s->surf[i];
        if (spec_only && !surf_is_specular(s, i)) continue;
        if (f->kind == 0) {
            v3 oc = sub(o, vf(f->center));
            double b = dot(oc, d), c = dot(oc, oc) - (double)f->radius * f->radius;
            double disc = b * b - c;
            if (disc < 0.0) continue;
            double sq = sqrt(disc);
            double ts[2] = {-b - sq, -b + sq};
            for (int j = 0; j < 2; j++)
                if (ts[j] > tmin && ts[j] < best->t) { best->t = ts[j]; best->prim = -1; best->surf = i; break; }
        } else if (f->kind == 1) {
            double t = tri_isect(o, d, vf(f->origin), vf(f->edge_u), vf(f->edge_v), NULL, NULL, 1);
            if (t > tmin && t < best->t) { best->t = t; best->prim = -1; best->surf = i; }
        }
    }
}

static void isect_tri(const orc_scene *s, int t, v3 o, v3 d, double tmin, int spec_only, hit_t *best) {
    int sid = s->TS[t];
    if (spec_only && !surf_is_specular(s, sid)) return;
    v3 v0 = vtx(s, s->I[3 * t]), v1 = vtx(s, s->I[3 * t + 1]), v2 = vtx(s, s->I[3 * t + 2]);
    double th = tri_isect(o, d, v0, sub(v1, v0), sub(v2, v0), NULL, NULL, 0);
    if (th > tmin && th < best->t) { best->t = th; best->prim = t; best->surf = sid; }
}

static int box_hit(const bnode *n, v3 o, v3 inv, double tmin, double tmax) {
    double t0 = tmin, t1 = tmax;
    for (int a = 0; a < 3; a++) {
        double oa = vget(o, a), ia = vget(inv, a);
        double ta = (n->lo[a] - oa) * ia, tb = (n->hi[a] - oa) * ia;
        if (ta != ta) ta = -1e300; /* 0*inf */
        if (tb != tb) tb = 1e300;
        if (ta > tb) { double x = ta; ta = tb; tb = x; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t0 > t1) return 0;
    }
    return 1;
}

/* closest hit with t in (tmin, tmax); use_bvh=0 is the brute-force pin */
static hit_t closest(const orc_scene *s, v3 o, v3 d, double tmin, double tmax, int spec_only, int use_bvh) {
    hit_t best; best.t = tmax; best.prim = -2; best.surf = -1; best.p = V(0, 0, 0);
    isect_analytic(s, o, d, tmin, spec_only, &best);
    if (s->n_tri > 0) {
        if (!use_bvh) {
            for (int t = 0; t < s->n_tri; t++) isect_tri(s, t, o, d, tmin, spec_only, &best);
        } else {
            v3 inv = V(1.0 / d.x, 1.0 / d.y, 1.0 / d.z);
            int stack[128], sp = 0;
            stack[sp++] = 0;
            while (sp > 0) {
                const bnode *n = &s->nodes[stack[--sp]];
                if (!box_hit(n, o, inv, tmin, best.t)) continue;
                if (n->left < 0) {
                    for (int j = n->first; j < n->first + n->count; j++) isect_tri(s, s->order[j], o, d, tmin, spec_only, &best);
                } else {
                    stack[sp++] = n->left;
                    stack[sp++] = n->right;
                }
            }
        }
    }
    if (best.surf >= 0) best.p = add(o, mul(d, best.t));
    return best;
}

/* ------------------------------------------------------------------------ */
/* local geometry at a vertex                                                 */
/* ------------------------------------------------------------------------ */
/* a chain vertex; (oa, ob): the offset normal's slopes in the vertex's shading frame
 * (s, t, n) for a glossy surface, 0 for a pure specular one [R37] */
typedef struct { v3 p; int prim, surf; double oa, ob; } cvtx;

/* glossy chains: "we sample the offset normal from the microfacet distribution
 * before manifold sampling" -- GGX(alpha) normals m by D(m) cos(theta_m):
 * tan(theta_m) = alpha sqrt(u1 / (1 - u1)), phi_m = 2 pi u2; slopes m_x/m_z, m_y/m_z [R37] */
static void ggx_slopes(double alpha, double u1, double u2, double *a, double *b) {
    if (!(alpha > 0.0)) { *a = *b = 0.0; return; }
    double tt = alpha * sqrt(u1 / (1.0 - u1));
    double ph = 6.28318530717958647692 * u2;
    *a = tt * cos(ph);
    *b = tt * sin(ph);
}

/* geometric normal (outward [R9]) */
static v3 geo_normal(const orc_scene *s, const cvtx *x) {
    const orc_surface *f = &s->surf[x->surf];
    if (f->kind == 0) return nrmz(sub(x->p, vf(f->center)));
    if (f->kind == 1) return nrmz(cross(vf(f->edge_u), vf(f->edge_v)));
    int t = x->prim;
    v3 v0 = vtx(s, s->I[3 * t]), v1 = vtx(s, s->I[3 * t + 1]), v2 = vtx(s, s->I[3 * t + 2]);
    return nrmz(cross(sub(v1, v0), sub(v2, v0)));
}

/* shading normal n_s and, for a tangent displacement v, its derivative d_v n_s.
 * mesh: Phong interpolation n = n~/|n~|, n~ = sum b_j n_j (BASELINE.json configs[1]
 * "interpolated vertex normals"); derivative from the barycentric gradient [R3]. */
static v3 shading_normal(const orc_scene *s, const cvtx *x, int nv, const v3 *vs, v3 *dns) {
    const orc_surface *f = &s->surf[x->surf];
    if (f->kind == 0) {
        v3 r = sub(x->p, vf(f->center));
        double rl = len(r);
        v3 n = mul(r, 1.0 / rl);
        for (int j = 0; j < nv; j++) dns[j] = mul(sub(vs[j], mul(n, dot(n, vs[j]))), 1.0 / rl);
        return n;
    }
    if (f->kind == 1) {
        for (int j = 0; j < nv; j++) dns[j] = V(0, 0, 0);
        return nrmz(cross(vf(f->edge_u), vf(f->edge_v)));
    }
    int t = x->prim;
    int i0 = s->I[3 * t], i1 = s->I[3 * t + 1], i2 = s->I[3 * t + 2];
    v3 v0 = vtx(s, i0), e1 = sub(vtx(s, i1), v0), e2 = sub(vtx(s, i2), v0);
    v3 Ng = cross(e1, e2);
    double nn = dot(Ng, Ng);
    v3 r = sub(x->p, v0);
    double b1 = dot(cross(r, e2), Ng) / nn, b2 = dot(cross(e1, r), Ng) / nn, b0 = 1.0 - b1 - b2;
    v3 n0 = vnr(s, i0), n1 = vnr(s, i1), n2 = vnr(s, i2);
    v3 nt = add(add(mul(n0, b0), mul(n1, b1)), mul(n2, b2));
    double nl = len(nt);
    v3 n = mul(nt, 1.0 / nl);
    for (int j = 0; j < nv; j++) {
        double db1 = dot(cross(vs[j], e2), Ng) / nn, db2 = dot(cross(e1, vs[j]), Ng) / nn;
        v3 dnt = add(mul(sub(n1, n0), db1), mul(sub(n2, n0), db2));
        dns[j] = mul(sub(dnt, mul(n, dot(n, dnt))), 1.0 / nl);
    }
    return n;
}

/* ------------------------------------------------------------------------ */
/* specular constraint at vertex i (generalized half vector, [R1][R2])        */
/* ------------------------------------------------------------------------ */
typedef struct {
    v3 wi, wo, h, n, s, t, ng, sg, tg;
    double li, lo, eta_i, eta_o, hlen;
    v3 dn[2]; /* d n_s along sg, tg */
    double oa, ob; /* offset slopes [R37] */
    int glossy;
} cterm;

/* returns 0 on a degenerate configuration */
static int cterm_eval(const orc_scene *sc, v3 a, const cvtx *x, v3 b, int isT, cterm *c) {
    const orc_surface *f = &sc->surf[x->surf];
    v3 da = sub(a, x->p), db = sub(b, x->p);
    c->li = len(da); c->lo = len(db);
    if (!(c->li > 0.0) || !(c->lo > 0.0)) return 0;
    c->wi = mul(da, 1.0 / c->li);
    c->wo = mul(db, 1.0 / c->lo);
    c->ng = geo_normal(sc, x);
    onb(c->ng, &c->sg, &c->tg); /* step parameterization [R4] */
    v3 vs[2] = {c->sg, c->tg};
    c->n = shading_normal(sc, x, 2, vs, c->dn);
    onb(c->n, &c->s, &c->t); /* constraint frame [R3] */
    if (isT) {
        int out = dot(c->wi, c->ng) > 0.0; /* media from the side of w_i [R9] */
        c->eta_i = out ? f->eta_out : f->eta_in;
        c->eta_o = out ? f->eta_in : f->eta_out;
    } else {
        c->eta_i = c->eta_o = 1.0;
    }
    v3 ht = add(mul(c->wi, c->eta_i), mul(c->wo, c->eta_o));
    c->hlen = len(ht);
    if (!(c->hlen > 0.0) || !isfinite(c->hlen)) return 0;
    c->h = mul(ht, 1.0 / c->hlen);
    c->oa = x->oa;
    c->ob = x->ob;
    c->glossy = f->roughness > 0.0f;
    return 1;
}

/* C_i = (s.h, t.h) (R1); with an offset normal m = (oa, ob, 1) in the frame (s, t, n), h must
 * be parallel to m: C_i = (s.h - oa n.h, t.h - ob n.h) [R37] */
static void cterm_C(const cterm *c, double C[2]) {
    double hn = dot(c->n, c->h);
    C[0] = dot(c->s, c->h) - c->oa * hn;
    C[1] = dot(c->t, c->h) - c->ob * hn;
}

/* dh for a change u of h~ : P_h u = (u - h(h.u))/|h~| */
static v3 dh_of(const cterm *c, v3 u) { return mul(sub(u, mul(c->h, dot(c->h, u))), 1.0 / c->hlen); }
/* P_i v, P_o v */
static v3 Pi(const cterm *c, v3 v) { return mul(sub(v, mul(c->wi, dot(c->wi, v))), 1.0 / c->li); }
static v3 Po(const cterm *c, v3 v) { return mul(sub(v, mul(c->wo, dot(c->wo, v))), 1.0 / c->lo); }

/* dC/d(x_{i-1}) along v  (block L) */
static void dC_da(const cterm *c, v3 v, double out[2]) {
    v3 dh = dh_of(c, mul(Pi(c, v), c->eta_i));
    out[0] = dot(c->s, dh) - c->oa * dot(c->n, dh); out[1] = dot(c->t, dh) - c->ob * dot(c->n, dh);
}
/* dC/d(x_{i+1}) along v  (block U, and D_L for the light) */
static void dC_db(const cterm *c, v3 v, double out[2]) {
    v3 dh = dh_of(c, mul(Po(c, v), c->eta_o));
    out[0] = dot(c->s, dh) - c->oa * dot(c->n, dh); out[1] = dot(c->t, dh) - c->ob * dot(c->n, dh);
}
/* dC/d(x_i) along basis vector j (block D); frame moves by minimal rotation [R3] */
static void dC_dp(const cterm *c, int j, double out[2]) {
    v3 v = j == 0 ? c->sg : c->tg;
    v3 u = sub(mul(Pi(c, v), -c->eta_i), mul(Po(c, v), c->eta_o));
    v3 dh = dh_of(c, u);
    double hn = dot(c->h, c->n);
    if (c->glossy) { /* exact frame derivative (onb_d) and the offset terms [R37] */
        v3 ds, dt;
        onb_d(c->n, c->dn[j], &ds, &dt);
        double dhn = dot(c->dn[j], c->h) + dot(c->n, dh);
        out[0] = dot(ds, c->h) + dot(c->s, dh) - c->oa * dhn;
        out[1] = dot(dt, c->h) + dot(c->t, dh) - c->ob * dhn;
        return;
    }
    out[0] = dot(c->s, dh) - hn * dot(c->s, c->dn[j]);
    out[1] = dot(c->t, dh) - hn * dot(c->t, c->dn[j]);
}

/* whole chain: C (2k) and dense J (2k x 2k, row-major); returns 0 if degenerate */
static int chain_system(const orc_scene *sc, int k, uint32_t tau, v3 xD, v3 xL, const cvtx *x, double *C, double *J,
                        cterm *terms) {
    int m = 2 * k;
    if (J) memset(J, 0, sizeof(double) * (size_t)(m * m));
    for (int i = 0; i < k; i++) {
        v3 a = i == 0 ? xD : x[i - 1].p;
        v3 b = i == k - 1 ? xL : x[i + 1].p;
        if (!cterm_eval(sc, a, &x[i], b, (tau >> i) & 1u, &terms[i])) return 0;
        cterm_C(&terms[i], C + 2 * i);
    }
    if (J) {
        for (int i = 0; i < k; i++) {
            double o2[2];
            for (int j = 0; j < 2; j++) {
                dC_dp(&terms[i], j, o2);
                J[(2 * i) * m + 2 * i + j] = o2[0];
                J[(2 * i + 1) * m + 2 * i + j] = o2[1];
                if (i > 0) {
                    v3 v = j == 0 ? terms[i - 1].sg : terms[i - 1].tg;
                    dC_da(&terms[i], v, o2);
                    J[(2 * i) * m + 2 * (i - 1) + j] = o2[0];
                    J[(2 * i + 1) * m + 2 * (i - 1) + j] = o2[1];
                }
                if (i < k - 1) {
                    v3 v = j == 0 ? terms[i + 1].sg : terms[i + 1].tg;
                    dC_db(&terms[i], v, o2);
                    J[(2 * i) * m + 2 * (i + 1) + j] = o2[0];
                    J[(2 * i + 1) * m + 2 * (i + 1) + j] = o2[1];
                }
            }
        }
    }
    for (int i = 0; i < m; i++) if (!isfinite(C[i])) return 0;
    return 1;
}

/* dense LU with partial pivoting; solves A X = B for nr right-hand sides
 * (B is m x nr row-major, overwritten by X). returns 0 if singular. */
static int lu_solve(double *A, int m, double *B, int nr) {
    for (int col = 0; col < m; col++) {
        int piv = col;
        for (int r = col + 1; r < m; r++) if (fabs(A[r * m + col]) > fabs(A[piv * m + col])) piv = r;
        if (!(fabs(A[piv * m + col]) > 0.0)) return 0;
        if (piv != col) {
            for (int c = 0; c < m; c++) { double t = A[col * m + c]; A[col * m + c] = A[piv * m + c]; A[piv * m + c] = t; }
            for (int c = 0; c < nr; c++) { double t = B[col * nr + c]; B[col * nr + c] = B[piv * nr + c]; B[piv * nr + c] = t; }
        }
        for (int r = col + 1; r < m; r++) {
            double f = A[r * m + col] / A[col * m + col];
            if (f == 0.0) continue;
            for (int c = col; c < m; c++) A[r * m + c] -= f * A[col * m + c];
            for (int c = 0; c < nr; c++) B[r * nr + c] -= f * B[col * nr + c];
        }
    }
    for (int r = m - 1; r >= 0; r--) {
        for (int c = 0; c < nr; c++) {
            double acc = B[r * nr + c];
            for (int j = r + 1; j < m; j++) acc -= A[r * m + j] * B[j * nr + c];
            B[r * nr + c] = acc / A[r * m + r];
        }
    }
    for (int i = 0; i < m * nr; i++) if (!isfinite(B[i])) return 0;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* the manifold walk: Newton + sequential ray-traced reprojection [R5-R7]    */
/* ------------------------------------------------------------------------ */
static double *g_beta_hist = NULL; /* debug: beta per iteration (orc_walk_trace) */
static int newton(const orc_scene *sc, const orc_opts *o, int k, uint32_t tau, v3 xD, v3 xL, cvtx *x, int *iters,
                  double eps, double *res_hist) {
    double C[2 * KMAX], J[4 * KMAX * KMAX], D[2 * KMAX];
    cterm terms[KMAX];
    double beta = o->beta0;
    int m = 2 * k;
    for (int it = 0;; it++) {
        *iters = it;
        if (!chain_system(sc, k, tau, xD, xL, x, C, J, terms)) return ST_DEGENERATE;
        double nrm = 0.0;
        for (int i = 0; i < m; i++) if (fabs(C[i]) > nrm) nrm = fabs(C[i]);
        if (res_hist) res_hist[it] = nrm;
        if (g_beta_hist) g_beta_hist[it] = beta;
        if (nrm < o->tol) return ST_CONVERGED;
        int mx = (k >= 3 && o->max_iters_long > 0) ? o->max_iters_long : o->max_iters;
        if (it == mx) return ST_MAXITER;
        for (int i = 0; i < m; i++) D[i] = -C[i];
        if (!lu_solve(J, m, D, 1)) return ST_DEGENERATE;
        /* proposed points q_i on the geometric tangent planes */
        cvtx y[KMAX];
        int ok = 1;
        v3 prev = xD;
        for (int i = 0; i < k && ok; i++) {
            v3 q = add(x[i].p, mul(add(mul(terms[i].sg, D[2 * i]), mul(terms[i].tg, D[2 * i + 1])), beta));
            v3 dir = sub(q, prev);
            double dl = len(dir);
            if (!(dl > 0.0)) { ok = 0; break; }
            dir = mul(dir, 1.0 / dl);
            hit_t h = closest(sc, prev, dir, eps, 1e300, 1, 1);
            if (h.surf < 0 || h.surf != x[i].surf) { ok = 0; break; }
            y[i].p = h.p; y[i].prim = h.prim; y[i].surf = h.surf;
            y[i].oa = x[i].oa; y[i].ob = x[i].ob; /* the offsets stay (same surface) [R37] */
            prev = h.p;
        }
        if (ok) { for (int i = 0; i < k; i++) x[i] = y[i]; beta = beta * 2.0 < 1.0 ? beta * 2.0 : 1.0; }
        else beta *= 0.5;
    }
}

/* sidedness per tau_i with the geometric normal [R8][R9] */
static int sides_ok(const orc_scene *sc, int k, uint32_t tau, v3 xD, v3 xL, const cvtx *x) {
    for (int i = 0; i < k; i++) {
        v3 a = i == 0 ? xD : x[i - 1].p, b = i == k - 1 ? xL : x[i + 1].p;
        v3 ng = geo_normal(sc, &x[i]);
        double di = dot(sub(a, x[i].p), ng), dd = dot(sub(b, x[i].p), ng);
        if ((tau >> i) & 1u) { if (!(di * dd < 0.0)) return 0; }
        else { if (!(di * dd > 0.0)) return 0; }
    }
    return 1;
}

/* V: any hit against all surfaces on every segment, t in (eps, len-eps) */
static int visible_chain(const orc_scene *sc, int k, v3 xD, v3 xL, const cvtx *x, double eps) {
    for (int j = 0; j <= k; j++) {
        v3 a = j == 0 ? xD : x[j - 1].p, b = j == k ? xL : x[j].p;
        v3 d = sub(b, a);
        double l = len(d);
        d = mul(d, 1.0 / l);
        hit_t h = closest(sc, a, d, eps, l - eps, 0, 1);
        if (h.surf >= 0) return 0;
    }
    return 1;
}

/* unpolarized dielectric Fresnel reflectance; eta1 = medium of incidence */
double orc_fresnel(double cos_i, double eta1, double eta2) {
    cos_i = fabs(cos_i);
    double st2 = (eta1 / eta2) * (eta1 / eta2) * (1.0 - cos_i * cos_i);
    if (st2 >= 1.0) return 1.0;
    double ct = sqrt(1.0 - st2);
    double rs = (eta1 * cos_i - eta2 * ct) / (eta1 * cos_i + eta2 * ct);
    double rp = (eta2 * cos_i - eta1 * ct) / (eta2 * cos_i + eta1 * ct);
    return 0.5 * (rs * rs + rp * rp);
}

/* kappa: product of Fresnel R / (1-F) T / conductor rho, times (eta_D/eta_L)^2 [R12] */
static double kappa_of(const orc_scene *sc, int k, uint32_t tau, v3 xD, v3 xL, const cvtx *x) {
    double kap = 1.0, etaD = 1.0, etaL = 1.0;
    for (int i = 0; i < k; i++) {
        const orc_surface *f = &sc->surf[x[i].surf];
        v3 a = i == 0 ? xD : x[i - 1].p, b = i == k - 1 ? xL : x[i + 1].p;
        v3 wi = nrmz(sub(a, x[i].p)), wo = nrmz(sub(b, x[i].p));
        v3 ng = geo_normal(sc, &x[i]);
        v3 dummy[1];
        v3 ns = shading_normal(sc, &x[i], 0, NULL, dummy);
        if (f->roughness > 0.0f) { /* Fresnel at the micro-normal (offset normal) [R37] */
            v3 s, t;
            onb(ns, &s, &t);
            ns = nrmz(add(ns, add(mul(s, x[i].oa), mul(t, x[i].ob))));
        }
        int out_i = dot(wi, ng) > 0.0, out_o = dot(wo, ng) > 0.0;
        double eta_wi = out_i ? f->eta_out : f->eta_in;
        double eta_wo = out_o ? f->eta_out : f->eta_in;
        if (i == 0) etaD = eta_wi;
        if (i == k - 1) etaL = eta_wo;
        if (f->mat == 0) kap *= f->reflectance;
        else {
            double eta_other = out_i ? f->eta_in : f->eta_out;
            double F = orc_fresnel(dot(wi, ns), eta_wi, eta_other);
            kap *= ((tau >> i) & 1u) ? (1.0 - F) : F;
        }
    }
    return kap * (etaD / etaL) * (etaD / etaL);
}

/* light-side axes: area light: orthonormal axes of its plane; point light: of the
 * plane orthogonal to x_L - x_k [R11] */
static void light_axes(const orc_light *L, v3 xL, v3 xk, v3 *l1, v3 *l2) {
    if (L->kind == 1) {
        v3 nl = nrmz(cross(vf(L->edge_u), vf(L->edge_v)));
        *l1 = nrmz(vf(L->edge_u));
        *l2 = nrmz(cross(nl, *l1));
    } else {
        onb(nrmz(sub(xL, xk)), l1, l2);
    }
}

/* analytic generalized geometric term (without V): G = |n_D.w| |det dw_D/dA_L| [R11] */
static double ggt_analytic(const orc_scene *sc, int k, uint32_t tau, v3 xD, v3 nD, v3 xL, const orc_light *L,
                           const cvtx *x) {
    double C[2 * KMAX], J[4 * KMAX * KMAX], B[2 * KMAX * 2];
    cterm terms[KMAX];
    int m = 2 * k;
    if (!chain_system(sc, k, tau, xD, xL, x, C, J, terms)) return 0.0;
    v3 l1, l2;
    light_axes(L, xL, x[k - 1].p, &l1, &l2);
    memset(B, 0, sizeof(B));
    double d0[2], d1[2];
    dC_db(&terms[k - 1], l1, d0);
    dC_db(&terms[k - 1], l2, d1);
    B[(m - 2) * 2 + 0] = -d0[0]; B[(m - 1) * 2 + 0] = -d0[1];
    B[(m - 2) * 2 + 1] = -d1[0]; B[(m - 1) * 2 + 1] = -d1[1];
    if (!lu_solve(J, m, B, 2)) return 0.0;
    v3 r = sub(x[0].p, xD);
    double rl = len(r);
    v3 w = mul(r, 1.0 / rl);
    v3 e1, e2;
    onb(w, &e1, &e2);
    double M[2][2];
    for (int c = 0; c < 2; c++) {
        v3 dx = add(mul(terms[0].sg, B[0 * 2 + c]), mul(terms[0].tg, B[1 * 2 + c]));
        v3 dw = mul(sub(dx, mul(w, dot(w, dx))), 1.0 / rl);
        M[0][c] = dot(e1, dw);
        M[1][c] = dot(e2, dw);
    }
    return fabs(dot(nD, w)) * fabs(M[0][0] * M[1][1] - M[0][1] * M[1][0]);
}

/* ------------------------------------------------------------------------ */
/* guide tables (histogram stand-in for Eqs. 10-13) [R20]                     */
/* W_b = E_b>0 ? max(1, floor(fp32(E_b/E_max) * 2^20)) : 0;                    */
/* W'_b = sum W + nbins*W_b  (= 1/2 uniform + 1/2 learned, Eq. 13, alpha=1/2)  */
/* empty cell -> uniform ("learned component is absent")          */
/* ------------------------------------------------------------------------ */
void orc_guide_tables(const float *E, int n_cells, int n_bins, uint64_t *prefix) {
    for (int c = 0; c < n_cells; c++) {
        const float *e = E + (size_t)c * n_bins;
        float emax = 0.0f;
        for (int b = 0; b < n_bins; b++) if (e[b] > emax) emax = e[b];
        uint64_t sumW = 0;
        uint32_t *W = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n_bins);
        for (int b = 0; b < n_bins; b++) {
            uint32_t wb = 0;
            if (e[b] > 0.0f && emax > 0.0f) {
                float r = e[b] / emax;
                float q = floorf(r * 1048576.0f);
                wb = (uint32_t)q;
                if (wb < 1u) wb = 1u;
            }
            W[b] = wb;
            sumW += wb;
        }
        uint64_t acc = 0;
        for (int b = 0; b < n_bins; b++) {
            uint64_t wp = sumW == 0 ? 1u : sumW + (uint64_t)n_bins * W[b];
            acc += wp;
            prefix[(size_t)c * n_bins + b] = acc;
        }
        free(W);
    }
}

/* ------------------------------------------------------------------------ */
/* seeds: fp32, no contraction [R23]                                          */
/* ------------------------------------------------------------------------ */
static void onb_f(const float n[3], float b1[3], float b2[3]) {
    float sign = copysignf(1.0f, n[2]);
    float a = -1.0f / (sign + n[2]);
    float b = n[0] * n[1] * a;
    b1[0] = 1.0f + sign * n[0] * n[0] * a; b1[1] = sign * b; b1[2] = -sign * n[0];
    b2[0] = b; b2[1] = sign + n[1] * n[1] * a; b2[2] = -n[1];
}

/* light sample (purpose 0, trial 0) [R15] */
static void sample_light(const orc_scene *sc, const orc_opts *o, uint64_t walk, float xL[3], double *pdf, int *lid) {
    uint32_t r[4];
    draw(o, walk, 0u, 0u, r);
    int li = sc->n_light > 1 ? (int)uidx(r[2], (uint32_t)sc->n_light) : 0;
    const orc_light *L = &sc->light[li];
    *lid = li;
    if (L->kind == 1) {
        float a = u01(r[0]) - 0.5f, b = u01(r[1]) - 0.5f;
        for (int j = 0; j < 3; j++) xL[j] = L->position[j] + (a * L->edge_u[j] + b * L->edge_v[j]);
        double area = len(cross(vf(L->edge_u), vf(L->edge_v)));
        *pdf = 1.0 / (area * sc->n_light);
    } else {
        for (int j = 0; j < 3; j++) xL[j] = L->position[j];
        *pdf = 1.0 / sc->n_light;
    }
}

/* seed draw result: the deduction ray x_D -> tgt gives x_1 (Eq. 6); n = chain
 * length, tau = type string (learned/fixed) or init_bits (initializer: R/T per
 * dielectric vertex chosen while tracing), Pn = P(n) of the length mixture. */
typedef struct { float tgt[3]; int32_t bin; int n; uint32_t tau; int learned; uint32_t init_bits; double Pn; } seed_res;

static const uint32_t P0_INT[6] = {20, 20, 20, 20, 20, 19}; /* P_0(n) = (1,1,1,1,1,0.95)/5.95 [R22] */

static uint64_t mulhi_u64(uint32_t x, uint64_t S) { /* floor(x*S/2^32), exact */
    uint64_t X = x;
    return X * (S >> 32) + ((X * (S & 0xffffffffu)) >> 32);
}

static int guide_cell(const orc_seed_cfg *cfg, const float xD[3]) {
    int cx = (int)floorf(((xD[0] - cfg->grid_origin[0]) * (float)cfg->cells_x) / cfg->grid_extent[0]);
    int cz = (int)floorf(((xD[2] - cfg->grid_origin[1]) * (float)cfg->cells_y) / cfg->grid_extent[1]);
    if (cx < 0) cx = 0;
    if (cx > cfg->cells_x - 1) cx = cfg->cells_x - 1;
    if (cz < 0) cz = 0;
    if (cz > cfg->cells_y - 1) cz = cfg->cells_y - 1;
    return cz * cfg->cells_x + cx;
}

typedef struct { float split; int32_t axis, child[2]; } orc_snode; /* child >= 0 inner node, < 0 ~leaf */
static float canon0(float x) { return x + 0.0f; } /* -0 -> +0: one ordering of equal keys [R29] */

/* w_D ~ vMF(mu, kappa) on S^2 (Eq. 12, density kappa/(4 pi sinh kappa) e^{kappa mu.w}):
 * cos theta by the inverse CDF F(c) = (e^{kappa c} - e^{-kappa}) / (2 sinh kappa), written as
 * c = 1 + log(xi + (1 - xi) e^{-2 kappa}) / kappa with xi = 1 - u1 in (0, 1]; phi = 2 pi u2 [R31] */
static void vmf_dir(const float mu[3], float kap, float u1, float u2, float out[3]) {
    float xi = 1.0f - u1;
    float e2k = expf(-2.0f * kap);
    float ct = 1.0f + logf(xi + (1.0f - xi) * e2k) / kap;
    if (ct < -1.0f) ct = -1.0f;
    if (ct > 1.0f) ct = 1.0f;
    float st2 = 1.0f - ct * ct;
    float st = sqrtf(st2 > 0.0f ? st2 : 0.0f);
    float phi = 6.28318530717958647692f * u2;
    float cp = cosf(phi), sp = sinf(phi);
    float b1[3], b2[3];
    onb_f(mu, b1, b2);
    for (int j = 0; j < 3; j++) out[j] = ct * mu[j] + st * (cp * b1[j] + sp * b2[j]);
}

static int seed_target(const orc_scene *sc, const orc_seed_cfg *cfg, const orc_opts *o, uint64_t walk, uint32_t trial,
                       const float xD[3], const float xL[3], seed_res *sr) {
    uint32_t r[4];
    float *tgt = sr->tgt;
    int32_t *bin = &sr->bin;
    *bin = -1;
    sr->n = cfg->k;
    sr->tau = cfg->tau;
    sr->learned = 1;
    sr->init_bits = 0;
    sr->Pn = 1.0;
    if (cfg->mode == 0) { /* uniform on the sphere cap visible from x_D [R21-cfg0] */
        const orc_surface *f = &sc->surf[cfg->surf_id];
        float d[3] = {xD[0] - f->center[0], xD[1] - f->center[1], xD[2] - f->center[2]};
        float L = sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        float a[3] = {d[0] / L, d[1] / L, d[2] / L};
        float cmin = f->radius / L;
        draw(o, walk, 2u, trial, r);
        float u1 = u01(r[0]), u2 = u01(r[1]);
        float ct = 1.0f - u1 * (1.0f - cmin);
        float st2 = 1.0f - ct * ct;
        float st = sqrtf(st2 > 0.0f ? st2 : 0.0f);
        float phi = 6.28318530717958647692f * u2;
        float cp = cosf(phi), sp = sinf(phi);
        float b1[3], b2[3];
        onb_f(a, b1, b2);
        for (int j = 0; j < 3; j++) {
            float dir = ct * a[j] + st * (cp * b1[j] + sp * b2[j]);
            tgt[j] = f->center[j] + f->radius * dir;
        }
        return 1;
    }
    if (cfg->mode == 1) { /* triangle uniform by count among front-facing, rejection <= 32 [R21-cfg1] */
        const orc_surface *f = &sc->surf[cfg->surf_id];
        int tri = -1;
        for (uint32_t rr = 0; rr < 32u; rr++) {
            draw(o, walk, 16u + rr, trial, r);
            int t = f->tri_begin + (int)uidx(r[0], (uint32_t)f->tri_count);
            const double *P = sc->P;
            float v0[3], v1[3], v2[3];
            for (int j = 0; j < 3; j++) {
                v0[j] = (float)P[3 * sc->I[3 * t] + j];
                v1[j] = (float)P[3 * sc->I[3 * t + 1] + j];
                v2[j] = (float)P[3 * sc->I[3 * t + 2] + j];
            }
            float e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
            float e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
            float ng[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
            float dd[3] = {xD[0] - v0[0], xD[1] - v0[1], xD[2] - v0[2]};
            float fdot = dd[0] * ng[0] + dd[1] * ng[1] + dd[2] * ng[2];
            if (fdot > 0.0f) { tri = t; break; }
        }
        if (tri < 0) return 0;
        *bin = tri;
        draw(o, walk, 2u, trial, r);
        float u1 = u01(r[0]), u2 = u01(r[1]);
        float sq = sqrtf(u1);
        float b1 = sq * (1.0f - u2), b2 = sq * u2;
        for (int j = 0; j < 3; j++) {
            float v0 = (float)sc->P[3 * sc->I[3 * tri] + j];
            float e1 = (float)sc->P[3 * sc->I[3 * tri + 1] + j] - v0;
            float e2 = (float)sc->P[3 * sc->I[3 * tri + 2] + j] - v0;
            tgt[j] = v0 + (b1 * e1 + b2 * e2);
        }
        return 1;
    }
    if (cfg->mode == 2) { /* guided bin over surface (u,v) via integer CDF [R20] */
        int nb = cfg->bins_x * cfg->bins_y;
        const uint64_t *pf = cfg->prefix + (size_t)guide_cell(cfg, xD) * nb;
        uint64_t S = pf[nb - 1];
        draw(o, walk, 1u, trial, r);
        uint64_t t = mulhi_u64(r[0], S); /* floor(x*S/2^32) */
        int b = 0;
        while (pf[b] <= t) b++; /* upper_bound: first prefix > t */
        *bin = b;
        int bx = b % cfg->bins_x, by = b / cfg->bins_x;
        draw(o, walk, 2u, trial, r);
        float u = ((float)bx + u01(r[0])) / (float)cfg->bins_x;
        float v = ((float)by + u01(r[1])) / (float)cfg->bins_y;
        tgt[0] = cfg->uv_origin[0] + u * cfg->uv_scale[0];
        tgt[1] = cfg->uv_plane_y;
        tgt[2] = cfg->uv_origin[1] + v * cfg->uv_scale[1];
        return 1;
    }
    if (cfg->mode == 3 || cfg->mode == 4) {
        /* configs[4]: n ~ 1/2 P_0 + 1/2 P_e (Eqs. 10, 13), then one-sample MIS of the initializer
           and the learned (tau, w_D) (Eqs. 8, 11, 13) [R22].  mode 3: P_e from the histogram cell
           of x_D, w_D from its direction bins; mode 4: P_e from the STree leaf of
           (x_D, x_L), w_D from the leaf's vMF mixture of type tau (Eq. 12) [R28-R31] */
        int c;
        if (cfg->mode == 3) {
            c = guide_cell(cfg, xD);
        } else {
            const orc_snode *nodes = (const orc_snode *)cfg->nodes;
            float p[6] = {canon0(xD[0]), canon0(xD[1]), canon0(xD[2]), canon0(xL[0]), canon0(xL[1]), canon0(xL[2])};
            int ref = cfg->root_ref;
            while (ref >= 0) ref = p[nodes[ref].axis] < nodes[ref].split ? nodes[ref].child[0] : nodes[ref].child[1];
            c = ~ref;
            /* selective activation: no own sample in the leaf -> path tracing [R36] */
            if (o->selective && cfg->leaf_own && cfg->leaf_own[c] == 0) return -1;
        }
        const uint64_t *npf = cfg->n_prefix + (size_t)c * 6;
        draw(o, walk, 1u, 0u, r); /* n reused by every trial */
        uint64_t S = npf[5];
        uint64_t t = mulhi_u64(r[0], S);
        int n = 0;
        while (npf[n] <= t) n++;
        sr->n = n + 1;
        sr->Pn = (double)(npf[n] - (n > 0 ? npf[n - 1] : 0)) / (double)S;
        draw(o, walk, 1u, trial, r);
        int g0 = (1 << sr->n) - 2, gn = 1 << sr->n;
        const uint64_t *tpf = cfg->type_prefix + (size_t)c * 126 + g0;
        uint64_t Wg = tpf[gn - 1];
        float u, v;
        if (Wg > 0 && (r[1] >> 31)) {
            uint64_t tt = mulhi_u64(r[2], Wg);
            int m = 0;
            while (tpf[m] <= tt) m++;
            sr->tau = (uint32_t)m;
            sr->learned = 1;
            if (cfg->mode == 4) { /* lobe i ~ W_i (Eq. 12 weights w_i), then w_D ~ vMF(mu_i, kappa_i) */
                int glo = cfg->grp_off[(size_t)c * 127 + g0 + m], ghi = cfg->grp_off[(size_t)c * 127 + g0 + m + 1];
                uint64_t Sl = cfg->lobe_prefix[ghi - 1];
                uint64_t tl = mulhi_u64(r[3], Sl);
                int b = glo;
                while (cfg->lobe_prefix[b] <= tl) b++;
                *bin = b;
                uint32_t r2[4];
                draw(o, walk, 2u, trial, r2);
                const float *mu = cfg->lobe_mu + 4 * (size_t)b;
                float w[3];
                vmf_dir(mu, mu[3], u01(r2[0]), u01(r2[1]), w);
                for (int j = 0; j < 3; j++) tgt[j] = xD[j] + w[j];
                return 1;
            }
            int nb = cfg->bins_x * cfg->bins_y;
            const uint32_t *dpf = cfg->dir_prefix + ((size_t)c * 126 + g0 + m) * nb;
            uint64_t Sd = dpf[nb - 1];
            uint64_t td = mulhi_u64(r[3], Sd);
            int b = 0;
            while (dpf[b] <= td) b++;
            *bin = b;
            uint32_t r2[4];
            draw(o, walk, 2u, trial, r2);
            u = ((float)(b % cfg->bins_x) + u01(r2[0])) / (float)cfg->bins_x;
            v = ((float)(b / cfg->bins_x) + u01(r2[1])) / (float)cfg->bins_y;
        } else {
            uint32_t r3[4];
            draw(o, walk, 3u, trial, r3);
            u = u01(r3[0]);
            v = u01(r3[1]);
            sr->learned = 0;
            sr->tau = 0;
            sr->init_bits = r3[2];
        }
        /* equal-area hemisphere about +y: u = cos(theta), v = (phi + pi)/(2 pi) */
        float st2 = 1.0f - u * u;
        float st = sqrtf(st2 > 0.0f ? st2 : 0.0f);
        float phi = 6.28318530717958647692f * v - 3.14159265358979323846f;
        float cp = cosf(phi), sp = sinf(phi);
        tgt[0] = xD[0] + st * cp;
        tgt[1] = xD[1] + u;
        tgt[2] = xD[2] + st * sp;
        return 1;
    }
    return 0;
}


/* deduction recursion Eq. 6 with s_R / s_T by tau [R14].
 * learned = 0 (initializer, "generated by ray tracing, deciding the
 * scattering type"): vertex i on a dielectric takes bit i of tau as T/R, a
 * conductor always R; the resolved string is returned in *tau_out [R22]. */
/* test hook: offset uniforms (u1, u2 per vertex) for the explicit-chain entry points
 * (orc_constraint, orc_newton_chain, orc_walk_from_target, orc_ggt, orc_kappa); NULL = 0 */
static const double *g_test_uv = NULL;
static double g_test_uv_buf[2 * KMAX];
void orc_set_offset_uv(const double *uv, int k) {
    if (!uv) { g_test_uv = NULL; return; }
    for (int i = 0; i < 2 * k && i < 2 * KMAX; i++) g_test_uv_buf[i] = uv[i];
    g_test_uv = g_test_uv_buf;
}
static void set_offsets(const orc_scene *sc, cvtx *x, int k, const double *uv) {
    for (int i = 0; i < k; i++) {
        if (uv) ggx_slopes(sc->surf[x[i].surf].roughness, uv[2 * i], uv[2 * i + 1], &x[i].oa, &x[i].ob);
        else x[i].oa = x[i].ob = 0.0;
    }
}
/* the walk's offset uniforms: vertex i takes words 2(i&1), 2(i&1)+1 of draw (11 + i/2, trial 0):
 * drawn once per walk and reused by every trial (the chains are "constrained to
 * this offset normal") [R37] */
static void walk_offset_uv(const orc_opts *o, uint64_t walk, int k, double *uv) {
    uint32_t r[4];
    for (int i = 0; i < k; i++) {
        if ((i & 1) == 0) draw(o, walk, 11u + (uint32_t)(i >> 1), 0u, r);
        uv[2 * i] = (double)u01(r[2 * (i & 1)]);
        uv[2 * i + 1] = (double)u01(r[2 * (i & 1) + 1]);
    }
}

static int deduce_ex(const orc_scene *sc, int k, uint32_t tau, int learned, v3 xD, v3 target, double eps, cvtx *x,
                     uint32_t *tau_out, const double *ouv) {
    uint32_t res = 0;
    v3 d = sub(target, xD);
    double dl = len(d);
    if (!(dl > 0.0)) return 0;
    d = mul(d, 1.0 / dl);
    v3 o = xD;
    for (int i = 0; i < k; i++) {
        hit_t h = closest(sc, o, d, eps, 1e300, 1, 1);
        if (h.surf < 0) return 0;
        x[i].p = h.p; x[i].prim = h.prim; x[i].surf = h.surf;
        x[i].oa = x[i].ob = 0.0;
        if (ouv) ggx_slopes(sc->surf[h.surf].roughness, ouv[2 * i], ouv[2 * i + 1], &x[i].oa, &x[i].ob);
        uint32_t bit = (tau >> i) & 1u;
        if (!learned && sc->surf[h.surf].mat == 0) bit = 0u;
        if (bit && sc->surf[h.surf].mat != 1) return 0; /* T on a conductor */
        res |= bit << i;
        if (i < k - 1) {
            const orc_surface *f = &sc->surf[h.surf];
            v3 ng = geo_normal(sc, &x[i]);
            v3 dummy[1];
            v3 n = shading_normal(sc, &x[i], 0, NULL, dummy);
            if (f->roughness > 0.0f) { /* scatter about the offset normal [R37] */
                v3 s, t;
                onb(n, &s, &t);
                n = nrmz(add(n, add(mul(s, x[i].oa), mul(t, x[i].ob))));
            }
            int outside = dot(d, ng) < 0.0;
            if (dot(d, n) > 0.0) n = mul(n, -1.0);
            double ci = -dot(d, n);
            if (!(ci > 0.0)) return 0;
            if (!bit) {
                d = add(d, mul(n, 2.0 * ci));
            } else {
                double e1 = outside ? f->eta_out : f->eta_in, e2 = outside ? f->eta_in : f->eta_out;
                double eta = e1 / e2;
                double k2 = 1.0 - eta * eta * (1.0 - ci * ci);
                if (k2 < 0.0) return 0; /* TIR */
                d = nrmz(add(mul(d, eta), mul(n, eta * ci - sqrt(k2))));
            }
        }
        o = h.p;
    }
    *tau_out = res;
    return 1;
}

static int deduce(const orc_scene *sc, int k, uint32_t tau, v3 xD, v3 target, double eps, cvtx *x) {
    uint32_t t2;
    return deduce_ex(sc, k, tau, 1, xD, target, eps, x, &t2, g_test_uv);
}

static int same_chain(int k, const cvtx *a, const cvtx *b, double eps) {
    for (int i = 0; i < k; i++) {
        if (a[i].surf != b[i].surf) return 0;
        if (len(sub(a[i].p, b[i].p)) >= eps) return 0;
    }
    return 1;
}

static double eps_ray(const orc_scene *sc, const orc_opts *o) { return o->ray_eps > 0.0 ? o->ray_eps : 1e-4 * sc->extent; }
static double eps_same(const orc_scene *sc, const orc_opts *o) { return o->same_chain_eps > 0.0 ? o->same_chain_eps : 1e-4 * sc->extent; }

/* one attempt: seed -> deduce -> Newton -> sides (O4-O7); *k, *tau: the chain type */
static int attempt(const orc_scene *sc, const orc_seed_cfg *cfg, const orc_opts *o, uint64_t walk, uint32_t trial,
                   const float xD[3], v3 xL, cvtx *x, int *iters, seed_res *sr, int *k, uint32_t *tau) {
    *iters = 0;
    *k = cfg->k;
    *tau = cfg->tau;
    float xLf[3] = {(float)xL.x, (float)xL.y, (float)xL.z}; /* exact: x_L was drawn in fp32 */
    const int sok = seed_target(sc, cfg, o, walk, trial, xD, xLf, sr);
    if (sok < 0) return ST_INACTIVE;
    if (!sok) return ST_SEED_FAIL;
    *k = sr->n;
    v3 xd = vf(xD);
    double eps = eps_ray(sc, o);
    double ouv[2 * KMAX];
    walk_offset_uv(o, walk, sr->n, ouv);
    if (!deduce_ex(sc, sr->n, sr->learned ? sr->tau : sr->init_bits, sr->learned, xd, vf(sr->tgt), eps, x, tau, ouv))
        return ST_SEED_FAIL;
    int st = newton(sc, o, *k, *tau, xd, xL, x, iters, eps, NULL);
    if (st == ST_CONVERGED && !sides_ok(sc, *k, *tau, xd, xL, x)) st = ST_BAD_SIDE;
    return st;
}

/* finish a converged chain: V, kappa, G, T (Eq. 2) */
static int finish(const orc_scene *sc, const orc_opts *o, int k, uint32_t tau, v3 xD, v3 nD, v3 xL, const orc_light *L,
                  const cvtx *x, double *G, double *T, double *kap) {
    *G = *T = *kap = 0.0;
    if (!visible_chain(sc, k, xD, xL, x, eps_ray(sc, o))) return ST_OCCLUDED;
    *kap = kappa_of(sc, k, tau, xD, xL, x);
    *G = ggt_analytic(sc, k, tau, xD, nD, xL, L, x);
    double Le = L->emit;
    if (L->kind == 1) { /* one-sided emitter */
        v3 nl = nrmz(cross(vf(L->edge_u), vf(L->edge_v)));
        if (!(dot(sub(x[k - 1].p, xL), nl) > 0.0)) Le = 0.0;
    }
    *T = *kap * *G * Le;
    return ST_CONVERGED;
}

/* The batched walk over explicit walk indices (walk = recv*spp + s).
 * Primary attempt (trial 0), then reciprocal-probability trials (Eq. 15):
 * first trial t whose converged, side-valid chain is same_chain(., x*) gives
 * k=t; w = T*k/(P(n)*pdf_L) with P(n)=1 for fixed-length configs [R13]. */
int orc_walks(const void *h, const orc_seed_cfg *cfg, const orc_opts *o, const float *xD, const float *nD, int32_t spp,
              const int64_t *walks, int64_t n, orc_walk_out *out) {
    const orc_scene *sc = (const orc_scene *)h;
    for (int64_t q = 0; q < n; q++) {
        orc_walk_out *r = &out[q];
        memset(r, 0, sizeof(*r));
        int64_t wi = walks[q];
        int64_t recv = wi / spp;
        uint64_t wid = o->walk_id_base + (uint64_t)wi;
        const float *xd = xD + 3 * recv, *nd = nD + 3 * recv;
        float xLf[3];
        int lid;
        sample_light(sc, o, wid, xLf, &r->pdfL, &lid);
        v3 xL = vf(xLf);
        r->xL[0] = xL.x; r->xL[1] = xL.y; r->xL[2] = xL.z;
        cvtx x[KMAX];
        int iters, k;
        uint32_t tau;
        seed_res sr;
        int st = attempt(sc, cfg, o, wid, 0u, xd, xL, x, &iters, &sr, &k, &tau);
        memcpy(r->target, sr.tgt, sizeof(sr.tgt));
        r->bin = sr.bin;
        r->k = k;
        r->tau = tau;
        r->Pn = sr.Pn;
        r->attempts = 1;
        r->iters = iters;
        r->total_iters = iters;
        if (st == ST_CONVERGED) st = finish(sc, o, k, tau, vf(xd), vf(nd), xL, &sc->light[lid], x, &r->G, &r->T, &r->kappa);
        r->status = st;
        if (st == ST_CONVERGED || st == ST_OCCLUDED || st == ST_BAD_SIDE || st == ST_MAXITER || st == ST_DEGENERATE) {
            for (int i = 0; i < k; i++) {
                r->pos[i][0] = x[i].p.x; r->pos[i][1] = x[i].p.y; r->pos[i][2] = x[i].p.z;
                r->prim[i] = x[i].prim; r->surf[i] = x[i].surf;
            }
        }
        if (st == ST_CONVERGED && r->T > 0.0 && o->trials) {
            /* R x M: repetition rep draws its trials with counter rep*2^20 + t [R32] */
            int M = o->recip_repeats > 1 ? o->recip_repeats : 1;
            uint32_t ksum = 0;
            double es = eps_same(sc, o);
            for (int rep = 0; rep < M; rep++) {
                uint32_t kk = 0;
                for (uint32_t t = 1; t <= o->k_max; t++) {
                    cvtx y[KMAX];
                    int it2, k2;
                    uint32_t tau2;
                    seed_res s2r;
                    int s2 = attempt(sc, cfg, o, wid, ((uint32_t)rep << 20) + t, xd, xL, y, &it2, &s2r, &k2, &tau2);
                    r->attempts++;
                    r->total_iters += it2;
                    if (s2 == ST_CONVERGED && k2 == k && tau2 == tau && same_chain(k, y, x, es)) { kk = t; break; }
                }
                if (kk == 0) { kk = o->k_max; r->truncated = 1; }
                ksum += kk;
            }
            r->trials = ksum;
            /* Eq. 15: w = T <1/P> / (P(n) pdf_L), <1/P> = mean of the M geometric counts */
            r->w = r->T * ((double)ksum / (double)M) / (r->Pn * r->pdfL);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* exports for pins                                                           */
/* ------------------------------------------------------------------------ */
/* closest hit: returns surf (-1 miss); t, prim, p */
int orc_closest(const void *h, const double o[3], const double d[3], double tmin, double tmax, int spec_only,
                int use_bvh, double *t, int32_t *prim, double p[3]) {
    hit_t r = closest((const orc_scene *)h, V(o[0], o[1], o[2]), V(d[0], d[1], d[2]), tmin, tmax, spec_only, use_bvh);
    *t = r.t; *prim = r.prim; p[0] = r.p.x; p[1] = r.p.y; p[2] = r.p.z;
    return r.surf;
}

/* constraint vector and dense Jacobian at an explicit chain */
int orc_constraint(const void *h, int k, uint32_t tau, const double xD[3], const double xL[3], const double *pos,
                   const int32_t *prim, const int32_t *surf, double *C, double *J) {
    cvtx x[KMAX];
    cterm terms[KMAX];
    for (int i = 0; i < k; i++) { x[i].p = V(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]); x[i].prim = prim[i]; x[i].surf = surf[i]; }
    set_offsets((const orc_scene *)h, x, k, g_test_uv);
    return chain_system((const orc_scene *)h, k, tau, V(xD[0], xD[1], xD[2]), V(xL[0], xL[1], xL[2]), x, C, J, terms);
}

/* Newton from an explicit chain (idempotence, quadratic convergence);
 * chain updated in place; res_hist[max_iters+1] gets ||C||_inf per iteration */
int orc_newton_chain(const void *h, const orc_opts *o, int k, uint32_t tau, const double xD[3], const double xL[3],
                     double *pos, int32_t *prim, int32_t *surf, int32_t *iters, double *res_hist) {
    const orc_scene *sc = (const orc_scene *)h;
    cvtx x[KMAX];
    for (int i = 0; i < k; i++) { x[i].p = V(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]); x[i].prim = prim[i]; x[i].surf = surf[i]; }
    set_offsets((const orc_scene *)h, x, k, g_test_uv);
    int it;
    int st = newton(sc, o, k, tau, V(xD[0], xD[1], xD[2]), V(xL[0], xL[1], xL[2]), x, &it, eps_ray(sc, o), res_hist);
    for (int i = 0; i < k; i++) { pos[3 * i] = x[i].p.x; pos[3 * i + 1] = x[i].p.y; pos[3 * i + 2] = x[i].p.z; prim[i] = x[i].prim; surf[i] = x[i].surf; }
    *iters = it;
    return st;
}

/* full single walk from an explicit seed target and x_L (no trials):
 * deduce -> Newton -> sides -> V -> kappa, G, T.  Used for basin maps. */
int orc_walk_from_target(const void *h, const orc_opts *o, int k, uint32_t tau, int light_id, const double xD[3],
                         const double nD[3], const double xL[3], const double target[3], double *pos, int32_t *prim,
                         int32_t *surf, int32_t *iters, double *G, double *T) {
    const orc_scene *sc = (const orc_scene *)h;
    cvtx x[KMAX];
    v3 xd = V(xD[0], xD[1], xD[2]), xl = V(xL[0], xL[1], xL[2]);
    double eps = eps_ray(sc, o), kap;
    *iters = 0; *G = *T = 0.0;
    if (!deduce(sc, k, tau, xd, V(target[0], target[1], target[2]), eps, x)) return ST_SEED_FAIL;
    int st = newton(sc, o, k, tau, xd, xl, x, iters, eps, NULL);
    if (st == ST_CONVERGED && !sides_ok(sc, k, tau, xd, xl, x)) st = ST_BAD_SIDE;
    if (st == ST_CONVERGED) st = finish(sc, o, k, tau, xd, V(nD[0], nD[1], nD[2]), xl, &sc->light[light_id], x, G, T, &kap);
    for (int i = 0; i < k; i++) { pos[3 * i] = x[i].p.x; pos[3 * i + 1] = x[i].p.y; pos[3 * i + 2] = x[i].p.z; prim[i] = x[i].prim; surf[i] = x[i].surf; }
    return st;
}

/* G at an explicit admissible chain: analytic (method=0) or finite-difference
 * re-convergence with step delta (method=1; test-only) */
double orc_ggt(const void *h, const orc_opts *o, int method, double delta, int k, uint32_t tau, int light_id,
               const double xD[3], const double nD[3], const double xL[3], const double *pos, const int32_t *prim,
               const int32_t *surf) {
    const orc_scene *sc = (const orc_scene *)h;
    cvtx x[KMAX];
    for (int i = 0; i < k; i++) { x[i].p = V(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]); x[i].prim = prim[i]; x[i].surf = surf[i]; }
    set_offsets((const orc_scene *)h, x, k, g_test_uv);
    v3 xd = V(xD[0], xD[1], xD[2]), nd = V(nD[0], nD[1], nD[2]), xl = V(xL[0], xL[1], xL[2]);
    const orc_light *L = &sc->light[light_id];
    if (method == 0) return ggt_analytic(sc, k, tau, xd, nd, xl, L, x);
    v3 l1, l2;
    light_axes(L, xl, x[k - 1].p, &l1, &l2);
    v3 ax[2] = {l1, l2};
    v3 dw[2];
    orc_opts oo = *o;
    oo.tol = 1e-13;
    oo.max_iters = 60;
    for (int a = 0; a < 2; a++) {
        v3 wpm[2];
        for (int sgn = 0; sgn < 2; sgn++) {
            cvtx y[KMAX];
            memcpy(y, x, sizeof(cvtx) * (size_t)k);
            v3 xl2 = add(xl, mul(ax[a], sgn ? -delta : delta));
            int it;
            int st = newton(sc, &oo, k, tau, xd, xl2, y, &it, eps_ray(sc, o), NULL);
            if (st != ST_CONVERGED) return -1.0;
            wpm[sgn] = nrmz(sub(y[0].p, xd));
        }
        dw[a] = mul(sub(wpm[0], wpm[1]), 0.5 / delta);
    }
    v3 w = nrmz(sub(x[0].p, xd)), e1, e2;
    onb(w, &e1, &e2);
    double M00 = dot(e1, dw[0]), M01 = dot(e1, dw[1]), M10 = dot(e2, dw[0]), M11 = dot(e2, dw[1]);
    return fabs(dot(nd, w)) * fabs(M00 * M11 - M01 * M10);
}

double orc_kappa(const void *h, int k, uint32_t tau, const double xD[3], const double xL[3], const double *pos,
                 const int32_t *prim, const int32_t *surf) {
    cvtx x[KMAX];
    for (int i = 0; i < k; i++) { x[i].p = V(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]); x[i].prim = prim[i]; x[i].surf = surf[i]; }
    set_offsets((const orc_scene *)h, x, k, g_test_uv);
    return kappa_of((const orc_scene *)h, k, tau, V(xD[0], xD[1], xD[2]), V(xL[0], xL[1], xL[2]), x);
}

/* seed draw only (light + target + bin) for walk/trial; returns 0 on failure */
int orc_seed(const void *h, const orc_seed_cfg *cfg, const orc_opts *o, const float *xD, int32_t spp, int64_t walk,
             uint32_t trial, float xL[3], double *pdfL, float tgt[3], int32_t *bin) {
    const orc_scene *sc = (const orc_scene *)h;
    int lid;
    uint64_t wid = o->walk_id_base + (uint64_t)walk;
    sample_light(sc, o, wid, xL, pdfL, &lid);
    seed_res sr;
    int ok = seed_target(sc, cfg, o, wid, trial, xD + 3 * (walk / spp), xL, &sr);
    memcpy(tgt, sr.tgt, sizeof(sr.tgt));
    *bin = sr.bin;
    return ok;
}

/* full seed draw (configs[4] tests): n, tau/init bits, learned flag, P(n) */
int orc_seed_ex(const void *h, const orc_seed_cfg *cfg, const orc_opts *o, const float *xD, int32_t spp, int64_t walk,
                uint32_t trial, float tgt[3], int32_t *bin, int32_t *n, uint32_t *tau, int32_t *learned,
                uint32_t *init_bits, double *Pn) {
    const orc_scene *sc = (const orc_scene *)h;
    seed_res sr;
    float xL[3];
    double pdfL;
    int lid;
    sample_light(sc, o, o->walk_id_base + (uint64_t)walk, xL, &pdfL, &lid);
    int ok = seed_target(sc, cfg, o, o->walk_id_base + (uint64_t)walk, trial, xD + 3 * (walk / spp), xL, &sr);
    memcpy(tgt, sr.tgt, sizeof(sr.tgt));
    *bin = sr.bin; *n = sr.n; *tau = sr.tau; *learned = sr.learned; *init_bits = sr.init_bits; *Pn = sr.Pn;
    return ok;
}

/* reflect / refract with the deduction's conventions (d along propagation) */
int orc_scatter(int isT, double eta1, double eta2, const double d[3], const double n[3], double out[3]) {
    v3 dd = V(d[0], d[1], d[2]), nn = V(n[0], n[1], n[2]);
    if (dot(dd, nn) > 0.0) nn = mul(nn, -1.0);
    double ci = -dot(dd, nn);
    v3 r;
    if (!isT) r = add(dd, mul(nn, 2.0 * ci));
    else {
        double eta = eta1 / eta2, k2 = 1.0 - eta * eta * (1.0 - ci * ci);
        if (k2 < 0.0) return 0;
        r = nrmz(add(mul(dd, eta), mul(nn, eta * ci - sqrt(k2))));
    }
    out[0] = r.x; out[1] = r.y; out[2] = r.z;
    return 1;
}

/* geometric tangent basis (s^g, t^g) of the step parameterization [R4] */
void orc_tangent_basis(const void *h, int32_t prim, int32_t surf, const double p[3], double sg[3], double tg[3]) {
    cvtx x;
    x.p = V(p[0], p[1], p[2]); x.prim = prim; x.surf = surf;
    v3 a, b;
    onb(geo_normal((const orc_scene *)h, &x), &a, &b);
    sg[0] = a.x; sg[1] = a.y; sg[2] = a.z;
    tg[0] = b.x; tg[1] = b.y; tg[2] = b.z;
}

/* debug: primary walk from an explicit target with per-iteration ||C||_inf and beta */
int orc_walk_trace(const void *h, const orc_opts *o, int k, uint32_t tau, const double xD[3], const double xL[3],
                   const double target[3], double *res_hist, double *beta_hist, int32_t *iters) {
    const orc_scene *sc = (const orc_scene *)h;
    cvtx x[KMAX];
    v3 xd = V(xD[0], xD[1], xD[2]), xl = V(xL[0], xL[1], xL[2]);
    double eps = eps_ray(sc, o);
    *iters = 0;
    if (!deduce(sc, k, tau, xd, V(target[0], target[1], target[2]), eps, x)) return ST_SEED_FAIL;
    g_beta_hist = beta_hist;
    int st = newton(sc, o, k, tau, xd, xl, x, iters, eps, res_hist);
    g_beta_hist = NULL;
    return st;
}

/* guide accumulation (Eq. 9; histogram stand-in R20): for walks with
 * status CONVERGED and w > 0, hist[cell(x_D)][bin(x_1*)] += w.  The cell uses the
 * same fp32 expression as the seed draw; the bin of x_1* = (x, z) in the (u,v)
 * map u = (x - uv_origin)/uv_scale, clamped.  x1 is given as float (the
 * reported chain position). */
void orc_accumulate(const orc_seed_cfg *cfg, const float *xD, int32_t spp, int64_t n, const int32_t *status,
                    const float *w, const float *x1, double *hist) {
    int nb = cfg->bins_x * cfg->bins_y;
    for (int64_t i = 0; i < n; i++) {
        if (status[i] != ST_CONVERGED || !(w[i] > 0.0f)) continue;
        const float *xd = xD + 3 * (i / spp);
        int cx = (int)floorf(((xd[0] - cfg->grid_origin[0]) * (float)cfg->cells_x) / cfg->grid_extent[0]);
        int cz = (int)floorf(((xd[2] - cfg->grid_origin[1]) * (float)cfg->cells_y) / cfg->grid_extent[1]);
        if (cx < 0) cx = 0;
        if (cx > cfg->cells_x - 1) cx = cfg->cells_x - 1;
        if (cz < 0) cz = 0;
        if (cz > cfg->cells_y - 1) cz = cfg->cells_y - 1;
        float u = (x1[3 * i] - cfg->uv_origin[0]) / cfg->uv_scale[0];
        float v = (x1[3 * i + 2] - cfg->uv_origin[1]) / cfg->uv_scale[1];
        int bx = (int)floorf(u * (float)cfg->bins_x), by = (int)floorf(v * (float)cfg->bins_y);
        if (bx < 0) bx = 0;
        if (bx > cfg->bins_x - 1) bx = cfg->bins_x - 1;
        if (by < 0) by = 0;
        if (by > cfg->bins_y - 1) by = cfg->bins_y - 1;
        hist[(size_t)(cz * cfg->cells_x + cx) * nb + by * cfg->bins_x + bx] += w[i];
    }
}

/* per-cell (or per-leaf) length and type tables from the per-type energies E[126] (R22):
 * W_n = E_n>0 ? max(1, floor(E_n/E_max 2^20)) : 0, n_prefix = cumsum(c_n sum W + 119 W_n)
 * (= 1/2 P_0 + 1/2 P_e, Eqs. 10, 13; no energy -> c_n); type weights per length group
 * likewise from E_tau (Eq. 11). */
static void typed_tables(const double *E, uint64_t *n_prefix, uint64_t *type_prefix) {
    double En[6], emax = 0.0;
    for (int n = 1; n <= 6; n++) {
        double e = 0.0;
        for (int m = 0; m < (1 << n); m++) e += E[(1 << n) - 2 + m];
        En[n - 1] = e;
        if (e > emax) emax = e;
    }
    uint64_t Wn[6], sumW = 0;
    for (int n = 0; n < 6; n++) {
        uint64_t w = 0;
        if (En[n] > 0.0 && emax > 0.0) {
            w = (uint64_t)floor((En[n] / emax) * 1048576.0);
            if (w < 1u) w = 1u;
        }
        Wn[n] = w;
        sumW += w;
    }
    uint64_t acc = 0;
    for (int n = 0; n < 6; n++) {
        acc += sumW == 0 ? P0_INT[n] : P0_INT[n] * sumW + 119u * Wn[n];
        n_prefix[n] = acc;
    }
    for (int n = 1; n <= 6; n++) {
        int g0 = (1 << n) - 2, gn = 1 << n;
        double gmax = 0.0;
        for (int m = 0; m < gn; m++) if (E[g0 + m] > gmax) gmax = E[g0 + m];
        uint64_t a2 = 0;
        for (int m = 0; m < gn; m++) {
            uint64_t w = 0;
            if (E[g0 + m] > 0.0 && gmax > 0.0) {
                w = (uint64_t)floor((E[g0 + m] / gmax) * 1048576.0);
                if (w < 1u) w = 1u;
            }
            a2 += w;
            type_prefix[g0 + m] = a2;
        }
    }
}

/* configs[4] guide tables from a typed direction histogram hist[cells][126][nb]
 * (R22): per (cell, type) energy E = sum of bins (fp64, bin order); per length
 * E_n = sum of its types (type order); W_n = E_n>0 ? max(1, floor(E_n/E_max 2^20)) : 0,
 * n_prefix = cumsum(c_n sum W + 119 W_n) (= 1/2 P_0 + 1/2 P_e, Eqs. 10, 13; empty
 * cell -> c_n); type weights per length group likewise from E_tau (Eq. 11);
 * direction weights per (cell, type) as R20 (fp32) but learned only. */
void orc_guide_dir_tables(const float *hist, int n_cells, int nb, uint64_t *n_prefix, uint64_t *type_prefix,
                          uint32_t *dir_prefix) {
    double *E = (double *)malloc(sizeof(double) * 126);
    for (int c = 0; c < n_cells; c++) {
        for (int t = 0; t < 126; t++) {
            const float *h = hist + ((size_t)c * 126 + t) * nb;
            double e = 0.0;
            float hmax = 0.0f;
            for (int b = 0; b < nb; b++) { e += (double)h[b]; if (h[b] > hmax) hmax = h[b]; }
            E[t] = e;
            uint32_t acc = 0;
            uint32_t *dp = dir_prefix + ((size_t)c * 126 + t) * nb;
            for (int b = 0; b < nb; b++) {
                uint32_t wb = 0;
                if (h[b] > 0.0f && hmax > 0.0f) {
                    float q = floorf((h[b] / hmax) * 1048576.0f);
                    wb = (uint32_t)q;
                    if (wb < 1u) wb = 1u;
                }
                acc += wb;
                dp[b] = acc;
            }
        }
        typed_tables(E, n_prefix + (size_t)c * 6, type_prefix + (size_t)c * 126);
    }
    free(E);
}

/* configs[4] accumulation: hist[cell(x_D)][type(n, tau)][bin(w_D*)] += w, bins of the
 * equal-area map u = cos(theta) (about +y), v = (atan2(w_z, w_x) + pi)/(2 pi) */
void orc_accumulate_dir(const orc_seed_cfg *cfg, const float *xD, int32_t spp, int64_t n, const int32_t *status,
                        const float *w, const float *x1, const int32_t *k, const uint32_t *tau, double *hist) {
    int nb = cfg->bins_x * cfg->bins_y;
    for (int64_t i = 0; i < n; i++) {
        if (status[i] != ST_CONVERGED || !(w[i] > 0.0f) || k[i] < 1 || k[i] > 6) continue;
        const float *xd = xD + 3 * (i / spp);
        int c = guide_cell(cfg, xd);
        float dx = x1[3 * i] - xd[0], dy = x1[3 * i + 1] - xd[1], dz = x1[3 * i + 2] - xd[2];
        float l = sqrtf(dx * dx + dy * dy + dz * dz);
        float u = dy / l;
        float v = (atan2f(dz, dx) + 3.14159265358979323846f) / 6.28318530717958647692f;
        int bu = (int)floorf(u * (float)cfg->bins_x), bv = (int)floorf(v * (float)cfg->bins_y);
        if (bu < 0) bu = 0;
        if (bu > cfg->bins_x - 1) bu = cfg->bins_x - 1;
        if (bv < 0) bv = 0;
        if (bv > cfg->bins_y - 1) bv = cfg->bins_y - 1;
        int type = (1 << k[i]) - 2 + (int)tau[i];
        hist[((size_t)c * 126 + type) * nb + bv * cfg->bins_x + bu] += w[i];
    }
}

/* ------------------------------------------------------------------------ */
/* STree + vMF guide, §5.5-5.6:                       */
/*   S = the sub-path samples of the last iteration (P:426 footnote)   */
/*   w = T <1/P> per sample (Eq. 9)                                */
/*   6D adaptive binary tree over (x_D, x_L), leaf threshold c sqrt|S|,       */
/*   eps k overlap copies, far samples discarded (P:518-523 + footnote)       */
/*   per leaf: P_e(n) (Eq. 10), P_e(tau|n) (Eq. 11), per type a vMF mixture   */
/*   with mu_i = w_D*_i, kappa_i = sigma_i^-2 from the nearest direction in   */
/*   the same (leaf, type) set, weights ~ w_i (Eq. 12)             */
/* Readings R28-R31.  Breadth-first: nodes and leaves are      */
/* numbered in the order they are created, level by level.                    */
/* ------------------------------------------------------------------------ */
typedef struct { float xD[3], xL[3], omega[3], w; int32_t type, pad; } orc_gsample; /* 48 B record */

typedef struct {
    int32_t n_nodes, n_leaves, root_ref, thr;
    int64_t n_valid, n_lobes;
    orc_snode *nodes;
    int64_t *leaf_begin, *leaf_count; /* into leaf_ids (the leaf's list, in its own order) */
    int64_t *leaf_ids;
    int32_t *grp_off;                 /* [leaves][127] */
    int64_t *lobe_sample;             /* [lobes] record index */
    uint64_t *lobe_prefix;            /* [lobes] */
    float *lobe_mu;                   /* [lobes][4] */
    uint64_t *n_prefix, *type_prefix; /* [leaves][6], [leaves][126] */
    int64_t *leaf_own;                /* [leaves] samples whose own key descends to the leaf [R36] */
} orc_stree;

static float skey(const orc_gsample *r, int a) { return canon0(a < 3 ? r->xD[a] : r->xL[a - 3]); }

/* stable sort of a node's list by one coordinate (equal coordinates keep the list's
 * order; the root list is in record order) [R29] -- a plain merge sort */
static void sort_by_axis(const orc_gsample *rec, int a, int64_t *ids, int64_t n, int64_t *tmp) {
    if (n < 2) return;
    int64_t h = n / 2;
    sort_by_axis(rec, a, ids, h, tmp);
    sort_by_axis(rec, a, ids + h, n - h, tmp);
    int64_t i = 0, j = h, k = 0;
    while (i < h && j < n) tmp[k++] = skey(rec + ids[j], a) < skey(rec + ids[i], a) ? ids[j++] : ids[i++];
    while (i < h) tmp[k++] = ids[i++];
    while (j < n) tmp[k++] = ids[j++];
    memcpy(ids, tmp, sizeof(int64_t) * n);
}

typedef struct { int64_t *ids; int64_t n; float lo[6], hi[6]; int depth; int parent, side; } orc_qnode;

void orc_stree_free(void *h) {
    orc_stree *t = (orc_stree *)h;
    if (!t) return;
    free(t->nodes); free(t->leaf_begin); free(t->leaf_count); free(t->leaf_ids); free(t->grp_off);
    free(t->lobe_sample); free(t->lobe_prefix); free(t->lobe_mu); free(t->n_prefix); free(t->type_prefix);
    free(t->leaf_own);
    free(t);
}

/* Build the guide from n records; a record is a sample iff w > 0 and 0 <= type < 126.
 * eps: overlap fraction (0.1, P:523 footnote); c_thr: threshold coefficient (1);
 * kappa = sigma'^-2 (Eq. 12), optionally clamped to [kappa_min, kappa_max]; the paper's
 * default is no clamp: kappa_min = 0, kappa_max = FLT_MAX (R30). */
void *orc_stree_build(const orc_gsample *rec, int64_t n, float eps, float c_thr, int32_t max_depth,
                      float kappa_min, float kappa_max) {
    orc_stree *t = (orc_stree *)calloc(1, sizeof(orc_stree));
    int64_t nv = 0;
    for (int64_t i = 0; i < n; i++) if (rec[i].w > 0.0f && rec[i].type >= 0 && rec[i].type < 126) nv++;
    t->n_valid = nv;
    /* threshold c sqrt|S| [R28]: floor in fp64 of c * sqrt(|S|), at least 1 */
    double thr_d = floor((double)c_thr * sqrt((double)nv));
    t->thr = thr_d < 1.0 ? 1 : (int32_t)thr_d;
    /* root: all samples in record order; box = fp32 min/max of their (x_D, x_L) */
    orc_qnode root;
    memset(&root, 0, sizeof(root));
    root.ids = (int64_t *)malloc(sizeof(int64_t) * (nv ? nv : 1));
    root.n = 0;
    for (int a = 0; a < 6; a++) { root.lo[a] = INFINITY; root.hi[a] = -INFINITY; }
    for (int64_t i = 0; i < n; i++) {
        if (!(rec[i].w > 0.0f && rec[i].type >= 0 && rec[i].type < 126)) continue;
        root.ids[root.n++] = i;
        for (int a = 0; a < 6; a++) {
            float x = skey(rec + i, a);
            if (x < root.lo[a]) root.lo[a] = x;
            if (x > root.hi[a]) root.hi[a] = x;
        }
    }
    int active[6], na = 0; /* split axes: those the samples span, in (x_D, x_L) order [R28] */
    for (int a = 0; a < 6; a++) if (nv > 0 && root.hi[a] > root.lo[a]) active[na++] = a;
    root.parent = -1;
    /* breadth-first queue */
    int64_t qcap = 1024, qh = 0, qt = 0;
    orc_qnode *q = (orc_qnode *)malloc(sizeof(orc_qnode) * qcap);
    q[qt++] = root;
    int64_t ncap = 64, lcap = 64, idcap = nv + 16, idn = 0;
    t->nodes = (orc_snode *)malloc(sizeof(orc_snode) * ncap);
    t->leaf_begin = (int64_t *)malloc(sizeof(int64_t) * lcap);
    t->leaf_count = (int64_t *)malloc(sizeof(int64_t) * lcap);
    t->leaf_ids = (int64_t *)malloc(sizeof(int64_t) * idcap);
    while (qh < qt) {
        orc_qnode nd = q[qh++];
        int ref;
        if (nd.n <= t->thr || nd.depth >= max_depth || na == 0) { /* leaf */
            if (t->n_leaves == lcap) {
                lcap *= 2;
                t->leaf_begin = (int64_t *)realloc(t->leaf_begin, sizeof(int64_t) * lcap);
                t->leaf_count = (int64_t *)realloc(t->leaf_count, sizeof(int64_t) * lcap);
            }
            if (idn + nd.n > idcap) {
                while (idn + nd.n > idcap) idcap *= 2;
                t->leaf_ids = (int64_t *)realloc(t->leaf_ids, sizeof(int64_t) * idcap);
            }
            memcpy(t->leaf_ids + idn, nd.ids, sizeof(int64_t) * nd.n);
            t->leaf_begin[t->n_leaves] = idn;
            t->leaf_count[t->n_leaves] = nd.n;
            idn += nd.n;
            ref = ~t->n_leaves++;
            free(nd.ids);
        } else { /* split at the midpoint of the cycled axis with eps k overlap [R28, R29] */
            if (t->n_nodes == ncap) { ncap *= 2; t->nodes = (orc_snode *)realloc(t->nodes, sizeof(orc_snode) * ncap); }
            int me = t->n_nodes++;
            ref = me;
            int a = active[nd.depth % na];
            float c = (nd.lo[a] + nd.hi[a]) * 0.5f;
            float delta = (nd.hi[a] - nd.lo[a]) * 0.25f; /* copies kept within half a child width */
            int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (nd.n ? nd.n : 1));
            sort_by_axis(rec, a, nd.ids, nd.n, tmp);
            free(tmp);
            int64_t m = 0;
            while (m < nd.n && skey(rec + nd.ids[m], a) < c) m++;
            int64_t e = (int64_t)floor((double)eps * (double)nd.n);
            int64_t eR = 0, eL = 0; /* the e nearest samples across the plane, the far ones dropped */
            while (eR < e && m + eR < nd.n && skey(rec + nd.ids[m + eR], a) - c <= delta) eR++;
            while (eL < e && m - 1 - eL >= 0 && c - skey(rec + nd.ids[m - 1 - eL], a) <= delta) eL++;
            /* samples inherited as copies that lie more than half a child width outside the child's
               box are far from it: discarded (P:523 footnote) [R29] */
            int64_t s0 = 0, s1 = nd.n;
            while (s0 < m && nd.lo[a] - skey(rec + nd.ids[s0], a) > delta) s0++;
            while (s1 > m && skey(rec + nd.ids[s1 - 1], a) - nd.hi[a] > delta) s1--;
            t->nodes[me].axis = a;
            t->nodes[me].split = c;
            t->nodes[me].child[0] = t->nodes[me].child[1] = 0;
            if (qt + 2 > qcap) {
                /* compact the consumed head, then grow */
                memmove(q, q + qh, sizeof(orc_qnode) * (qt - qh));
                qt -= qh; qh = 0;
                if (qt + 2 > qcap) { qcap *= 2; q = (orc_qnode *)realloc(q, sizeof(orc_qnode) * qcap); }
            }
            for (int side = 0; side < 2; side++) {
                orc_qnode ch;
                memcpy(ch.lo, nd.lo, sizeof(ch.lo));
                memcpy(ch.hi, nd.hi, sizeof(ch.hi));
                int64_t b0 = side == 0 ? s0 : m - eL, b1 = side == 0 ? m + eR : s1;
                if (side == 0) ch.hi[a] = c; else ch.lo[a] = c;
                ch.n = b1 - b0;
                ch.ids = (int64_t *)malloc(sizeof(int64_t) * (ch.n ? ch.n : 1));
                memcpy(ch.ids, nd.ids + b0, sizeof(int64_t) * ch.n);
                ch.depth = nd.depth + 1;
                ch.parent = me;
                ch.side = side;
                q[qt++] = ch;
            }
            free(nd.ids);
        }
        if (nd.parent < 0) t->root_ref = ref;
        else t->nodes[nd.parent].child[nd.side] = ref;
    }
    free(q);
    /* per leaf: lobes grouped by type (stable), kappa, weights, tables */
    int L = t->n_leaves;
    t->n_lobes = idn;
    t->grp_off = (int32_t *)malloc(sizeof(int32_t) * 127 * (size_t)L);
    t->lobe_sample = (int64_t *)malloc(sizeof(int64_t) * (idn ? idn : 1));
    t->lobe_prefix = (uint64_t *)malloc(sizeof(uint64_t) * (idn ? idn : 1));
    t->lobe_mu = (float *)malloc(sizeof(float) * 4 * (idn ? idn : 1));
    t->n_prefix = (uint64_t *)malloc(sizeof(uint64_t) * 6 * (size_t)L);
    t->type_prefix = (uint64_t *)malloc(sizeof(uint64_t) * 126 * (size_t)L);
    int64_t pos = 0;
    double E[126];
    for (int l = 0; l < L; l++) {
        const int64_t *ids = t->leaf_ids + t->leaf_begin[l];
        int64_t cnt = t->leaf_count[l];
        for (int ty = 0; ty < 126; ty++) {
            t->grp_off[(size_t)l * 127 + ty] = (int32_t)pos;
            int64_t g0 = pos;
            for (int64_t j = 0; j < cnt; j++) if (rec[ids[j]].type == ty) t->lobe_sample[pos++] = ids[j];
            /* E_tau = sum of w (Eqs. 10-11), in group order */
            double e = 0.0;
            float wmax = 0.0f;
            for (int64_t i = g0; i < pos; i++) {
                float wi = rec[t->lobe_sample[i]].w;
                e += (double)wi;
                if (wi > wmax) wmax = wi;
            }
            E[ty] = e;
            uint64_t acc = 0;
            for (int64_t i = g0; i < pos; i++) {
                const orc_gsample *ri = rec + t->lobe_sample[i];
                /* sigma_i: distance to the nearest other direction of the set (chord) [R30] */
                float d2min = INFINITY;
                for (int64_t j = g0; j < pos; j++) {
                    if (j == i) continue;
                    const orc_gsample *rj = rec + t->lobe_sample[j];
                    float dx = ri->omega[0] - rj->omega[0], dy = ri->omega[1] - rj->omega[1],
                          dz = ri->omega[2] - rj->omega[2];
                    float d2 = dx * dx + dy * dy + dz * dz;
                    if (d2 < d2min) d2min = d2;
                }
                /* Eq. 12: kappa = sigma'^-2; a lone lobe (no neighbour to measure a footprint,
                 * P:474 silent) takes kappa = 1; sigma' = 0 takes kappa_max [R30] */
                float kap = pos - g0 == 1 ? 1.0f : (d2min > 0.0f ? 1.0f / d2min : kappa_max);
                if (kap < kappa_min) kap = kappa_min;
                if (kap > kappa_max) kap = kappa_max;
                t->lobe_mu[4 * i] = ri->omega[0];
                t->lobe_mu[4 * i + 1] = ri->omega[1];
                t->lobe_mu[4 * i + 2] = ri->omega[2];
                t->lobe_mu[4 * i + 3] = kap;
                /* lobe weight ~ w_i, integer as R20 */
                float qf = floorf((ri->w / wmax) * 1048576.0f);
                uint64_t W = (uint64_t)qf;
                if (W < 1u) W = 1u;
                acc += W;
                t->lobe_prefix[i] = acc;
            }
        }
        t->grp_off[(size_t)l * 127 + 126] = (int32_t)pos;
        typed_tables(E, t->n_prefix + (size_t)l * 6, t->type_prefix + (size_t)l * 126);
    }
    /* selective activation [R36]: "samples (excluding those used for filtering)",
     * i.e. without the overlap copies, are the samples whose own key descends to the leaf */
    t->leaf_own = (int64_t *)calloc(t->n_leaves > 0 ? t->n_leaves : 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) {
        if (!(rec[i].w > 0.0f && rec[i].type >= 0 && rec[i].type < 126)) continue;
        int ref = t->root_ref;
        while (ref >= 0) ref = skey(rec + i, t->nodes[ref].axis) < t->nodes[ref].split ? t->nodes[ref].child[0]
                                                                                      : t->nodes[ref].child[1];
        t->leaf_own[~ref]++;
    }
    return t;
}

/* counts: n_nodes, n_leaves, root_ref, thr, n_valid, n_lobes */
void orc_stree_info(const void *h, int64_t out[6]) {
    const orc_stree *t = (const orc_stree *)h;
    out[0] = t->n_nodes; out[1] = t->n_leaves; out[2] = t->root_ref; out[3] = t->thr;
    out[4] = t->n_valid; out[5] = t->n_lobes;
}

/* copy out (caller sizes from orc_stree_info); any pointer may be NULL */
void orc_stree_get(const void *h, orc_snode *nodes, int64_t *leaf_begin, int64_t *leaf_count, int64_t *leaf_ids,
                   int32_t *grp_off, int64_t *lobe_sample, uint64_t *lobe_prefix, float *lobe_mu, uint64_t *n_prefix,
                   uint64_t *type_prefix, int64_t *leaf_own) {
    const orc_stree *t = (const orc_stree *)h;
    int64_t L = t->n_leaves, nl = t->n_lobes;
    if (nodes) memcpy(nodes, t->nodes, sizeof(orc_snode) * t->n_nodes);
    if (leaf_begin) memcpy(leaf_begin, t->leaf_begin, sizeof(int64_t) * L);
    if (leaf_count) memcpy(leaf_count, t->leaf_count, sizeof(int64_t) * L);
    if (leaf_ids) memcpy(leaf_ids, t->leaf_ids, sizeof(int64_t) * nl);
    if (grp_off) memcpy(grp_off, t->grp_off, sizeof(int32_t) * 127 * L);
    if (lobe_sample) memcpy(lobe_sample, t->lobe_sample, sizeof(int64_t) * nl);
    if (lobe_prefix) memcpy(lobe_prefix, t->lobe_prefix, sizeof(uint64_t) * nl);
    if (lobe_mu) memcpy(lobe_mu, t->lobe_mu, sizeof(float) * 4 * nl);
    if (n_prefix) memcpy(n_prefix, t->n_prefix, sizeof(uint64_t) * 6 * L);
    if (type_prefix) memcpy(type_prefix, t->type_prefix, sizeof(uint64_t) * 126 * L);
    if (leaf_own) memcpy(leaf_own, t->leaf_own, sizeof(int64_t) * L);
}

/* sample records from walk outputs (Eq. 9 samples of one iteration): x_D of the walk's receiver,
 * its x_L, w_D* = normalize(x_1* - x_D) (fp32), type = 2^n - 2 + tau, w; non-samples get w = 0 */
/* glossy separator (Eq. 14): w' = rho(w_v, w_D*) w with a microfacet lobe
 * rho = D(h) / (4 cos_v cos_D), D = GGX(alpha) = alpha^2 / (pi ((n.h)^2 (alpha^2 - 1) + 1)^2),
 * h = normalize(w_v + w_D*), w_v the receiver's unit direction towards the viewer [R35] */
static float separator_rho(const float n[3], const float wv[3], const float om[3], float alpha) {
    float cv = n[0] * wv[0] + n[1] * wv[1] + n[2] * wv[2];
    float cl = n[0] * om[0] + n[1] * om[1] + n[2] * om[2];
    if (!(cv > 0.0f) || !(cl > 0.0f)) return 0.0f;
    float hx = wv[0] + om[0], hy = wv[1] + om[1], hz = wv[2] + om[2];
    float hl = sqrtf(hx * hx + hy * hy + hz * hz);
    hx = hx / hl; hy = hy / hl; hz = hz / hl;
    float nh = n[0] * hx + n[1] * hy + n[2] * hz;
    float a2 = alpha * alpha;
    float t = nh * nh * (a2 - 1.0f) + 1.0f;
    float D = a2 / (3.14159265358979323846f * (t * t));
    return D / (4.0f * cv * cl);
}

void orc_record_samples(const float *xD, int32_t spp, int64_t n, const int32_t *status, const float *w,
                        const float *x1, const int32_t *k, const uint32_t *tau, const float *xL, const float *wv,
                        const float *nD, float alpha, orc_gsample *out) {
    for (int64_t i = 0; i < n; i++) {
        orc_gsample *r = out + i;
        memset(r, 0, sizeof(*r));
        const float *xd = xD + 3 * (i / spp);
        for (int j = 0; j < 3; j++) { r->xD[j] = xd[j]; r->xL[j] = xL[3 * i + j]; }
        r->type = -1;
        if (status[i] != ST_CONVERGED || !(w[i] > 0.0f) || k[i] < 1 || k[i] > 6) continue;
        float dx = x1[3 * i] - xd[0], dy = x1[3 * i + 1] - xd[1], dz = x1[3 * i + 2] - xd[2];
        float l = sqrtf(dx * dx + dy * dy + dz * dz);
        r->omega[0] = dx / l; r->omega[1] = dy / l; r->omega[2] = dz / l;
        r->type = (1 << k[i]) - 2 + (int32_t)tau[i];
        r->w = w[i];
        if (wv) { /* glossy separator: product weighting (Eq. 14) */
            r->w = w[i] * separator_rho(nD + 3 * (i / spp), wv + 3 * (i / spp), r->omega, alpha);
            if (!(r->w > 0.0f)) { r->w = 0.0f; r->type = -1; r->omega[0] = r->omega[1] = r->omega[2] = 0.0f; }
        }
    }
}

/* vMF direction draw as seed mode 4 does it (test export) */
void orc_vmf_sample(const float mu[3], float kap, float u1, float u2, float out[3]) { vmf_dir(mu, kap, u1, u2, out); }

/* ------------------------------------------------------------------------ */
/* Photon-based initial distribution: photons   */
/* traced from the emitters through the specular surfaces until they cross   */
/* the receiver plane; each landed photon with n >= 1 specular vertices is a */
/* sub-path sample (x_D, x_L, w_D*, type, w = its power) from which the      */
/* STree + vMF guide of iteration 0 is fitted instead of the empty guide.    */
/* Reading R33: emission, R/T by Fresnel, plane landing.         */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t n_photons;      /* N: power of a photon = n_light * Phi_light / N */
    uint64_t seed, photon_id_base;
    float plane_point[3], plane_normal[3]; /* receiver plane; photons land crossing it against the normal */
    int32_t max_vertices;   /* <= 6 */
    float ray_eps;          /* 0: 1e-4 * extent */
} orc_photon_desc;

/* one photon: record (w = 0, type = -1 if it does not land after >= 1 specular vertex);
 * nv, vertices (x_D order), prims, surfs for the pins */
static void trace_photon(const orc_scene *sc, const orc_photon_desc *pd, int64_t p, orc_gsample *rec, int *nv_out,
                         double *verts, int32_t *prims, int32_t *surfs) {
    orc_opts o;
    memset(&o, 0, sizeof(o));
    o.seed = pd->seed;
    uint64_t wid = pd->photon_id_base + (uint64_t)p;
    double eps = pd->ray_eps > 0.0f ? pd->ray_eps : 1e-4 * sc->extent;
    memset(rec, 0, sizeof(*rec));
    rec->type = -1;
    *nv_out = 0;
    uint32_t r[4];
    /* emission: light uniformly, position on it (as sample_light, purpose 8), direction (purpose 9) */
    draw(&o, wid, 8u, 0u, r);
    int li = sc->n_light > 1 ? (int)uidx(r[2], (uint32_t)sc->n_light) : 0;
    const orc_light *L = &sc->light[li];
    float xLf[3];
    double phi_light;
    v3 d;
    uint32_t q[4];
    draw(&o, wid, 9u, 0u, q);
    double u1 = (double)u01(q[0]), u2 = (double)u01(q[1]);
    double ph = 6.28318530717958647692 * u2;
    if (L->kind == 1) {
        float a = u01(r[0]) - 0.5f, b = u01(r[1]) - 0.5f;
        for (int j = 0; j < 3; j++) xLf[j] = L->position[j] + (a * L->edge_u[j] + b * L->edge_v[j]);
        v3 nl = cross(vf(L->edge_u), vf(L->edge_v));
        double area = len(nl);
        nl = mul(nl, 1.0 / area);
        phi_light = (double)L->emit * area * 3.14159265358979323846; /* Lambertian one-sided: L A pi */
        v3 b1, b2;
        onb(nl, &b1, &b2);
        double st = sqrt(u1), ct = sqrt(1.0 - u1);   /* cosine-weighted about n_L */
        d = add(mul(nl, ct), add(mul(b1, st * cos(ph)), mul(b2, st * sin(ph))));
    } else {
        for (int j = 0; j < 3; j++) xLf[j] = L->position[j];
        phi_light = 4.0 * 3.14159265358979323846 * (double)L->emit; /* isotropic point: 4 pi I */
        double z = 1.0 - 2.0 * u1, st = sqrt(fmax(0.0, 1.0 - z * z));
        d = V(st * cos(ph), z, st * sin(ph));
    }
    double w = (double)sc->n_light * phi_light / (double)pd->n_photons;
    v3 o3 = vf(xLf);
    v3 pp = vf(pd->plane_point), pn = nrmz(vf(pd->plane_normal));
    cvtx x[KMAX];
    int isT[KMAX];
    int nv = 0;
    uint32_t rt[4] = {0u, 0u, 0u, 0u};
    for (;;) {
        hit_t h = closest(sc, o3, d, eps, 1e300, 0, 1);
        double den = dot(d, pn);
        double tp = den < 0.0 ? dot(sub(pp, o3), pn) / den : -1.0;
        if (tp > eps && (h.surf < 0 || tp < h.t)) { /* lands on the receiver plane */
            if (nv >= 1) {
                v3 xd = add(o3, mul(d, tp));
                float xD[3] = {(float)xd.x, (float)xd.y, (float)xd.z};
                for (int j = 0; j < 3; j++) { rec->xD[j] = xD[j]; rec->xL[j] = xLf[j]; }
                float v1[3] = {(float)x[nv - 1].p.x, (float)x[nv - 1].p.y, (float)x[nv - 1].p.z};
                float dx = v1[0] - xD[0], dy = v1[1] - xD[1], dz = v1[2] - xD[2];
                float l = sqrtf(dx * dx + dy * dy + dz * dz);
                rec->omega[0] = dx / l; rec->omega[1] = dy / l; rec->omega[2] = dz / l;
                uint32_t tau = 0;
                for (int i = 0; i < nv; i++) tau |= (uint32_t)isT[nv - 1 - i] << i; /* x_D order */
                rec->type = (1 << nv) - 2 + (int32_t)tau;
                rec->w = (float)w;
                *nv_out = nv;
                for (int i = 0; i < nv; i++) {
                    const cvtx *v = &x[nv - 1 - i];
                    verts[3 * i] = v->p.x; verts[3 * i + 1] = v->p.y; verts[3 * i + 2] = v->p.z;
                    prims[i] = v->prim; surfs[i] = v->surf;
                }
            }
            return;
        }
        if (h.surf < 0 || nv == pd->max_vertices) return;      /* escaped, or chain too long */
        const orc_surface *f = &sc->surf[h.surf];
        if (f->mat == 2) return;                                  /* absorbed by a diffuse occluder */
        x[nv].p = h.p; x[nv].prim = h.prim; x[nv].surf = h.surf;
        v3 ng = geo_normal(sc, &x[nv]);
        v3 dummy[1];
        v3 n = shading_normal(sc, &x[nv], 0, NULL, dummy);
        int outside = dot(d, ng) < 0.0;
        if (dot(d, n) > 0.0) n = mul(n, -1.0);
        double ci = -dot(d, n);
        if (!(ci > 0.0)) return;
        int t = 0;
        /* vertex nv owns word nv&3 of draw (10, nv>>2), whatever its material [R33] */
        if ((nv & 3) == 0) draw(&o, wid, 10u, (uint32_t)(nv >> 2), rt);
        if (f->mat == 0) {
            w *= (double)f->reflectance;
        } else {                                                  /* R with probability F (Fresnel), else T */
            double e1 = outside ? f->eta_out : f->eta_in, e2 = outside ? f->eta_in : f->eta_out;
            double F = orc_fresnel(ci, e1, e2);
            t = (double)u01(rt[nv & 3]) >= F;
            if (t) {
                double eta = e1 / e2;
                double k2 = 1.0 - eta * eta * (1.0 - ci * ci);
                if (k2 < 0.0) return;
                d = nrmz(add(mul(d, eta), mul(n, eta * ci - sqrt(k2))));
            }
        }
        if (!t) d = add(d, mul(n, 2.0 * ci));
        isT[nv] = t;
        o3 = h.p;
        nv++;
    }
}

void orc_trace_photons(const void *h, const orc_photon_desc *pd, int64_t first, int64_t count, orc_gsample *rec,
                       int32_t *nv, double *verts, int32_t *prims, int32_t *surfs) {
    for (int64_t i = 0; i < count; i++) {
        int n_v = 0;
        double vv[3 * KMAX];
        int32_t pr[KMAX], su[KMAX];
        trace_photon((const orc_scene *)h, pd, first + i, rec + i, &n_v, vv, pr, su);
        if (nv) nv[i] = n_v;
        if (verts) memcpy(verts + 3 * KMAX * i, vv, sizeof(vv));
        if (prims) memcpy(prims + KMAX * i, pr, sizeof(pr));
        if (surfs) memcpy(surfs + KMAX * i, su, sizeof(su));
    }
}

/* ------------------------------------------------------------------------ */
/* online training schedule [R34], in passes:            */
/*   "We separate the training stage into several iterations with          */
/*    increasing budgets. Specifically, we double the sample count in each  */
/*    iteration. We stop the training stage immediately when 30% of the     */
/*    budget is already used. Besides, when a training iteration is         */
/*    finished, we start a new round if less than half of the training      */
/*    budget is used. Otherwise, we continue the current iteration until    */
/*    the rendering stage starts."                                          */
/* Simulated pass by pass: each pass belongs to the current iteration.      */
/* ------------------------------------------------------------------------ */
int orc_training_schedule(int64_t budget, double train_frac, int64_t *iters, int32_t max_iters, int64_t *render) {
    int64_t T = (int64_t)floor(train_frac * (double)budget); /* the training budget */
    int32_t m = 0;
    int64_t size = 1, in_cur = 0, used = 0;
    int extend = 0; /* the current iteration continues until training ends */
    while (used < T) {
        if (in_cur == 0) { if (m >= max_iters) return -1; iters[m++] = 0; }
        iters[m - 1]++; in_cur++; used++;
        if (!extend && in_cur == size && used < T) {      /* iteration finished */
            if (2 * used < T) { size *= 2; in_cur = 0; }   /* a new round */
            else extend = 1;                               /* continue the current one */
        }
    }
    *render = budget - T;
    return m;
}
