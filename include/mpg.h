/*
 * mpg.h -- C ABI of the B200-native batched manifold walk (libmpg.so).
 *
 * Method: Fan, Hong, Guo, Zou, Guo, Yan, "Manifold Path Guiding for Importance
 * Sampling Specular Chains", ACM TOG 42(6) 2023 (arXiv 2311.12818).
 * Citations "P:n" are lines of that paper's text; "Rn" are the
 * numbered readings of DESIGN.md §3 where the paper is silent.
 *
 * Conventions for every entry point
 *  - All functions return an mpg_status; on failure mpg_last_error() returns a
 *    thread-local message.  Argument errors are detected synchronously before
 *    anything is enqueued.  CUDA launch errors surface as MPG_ERR_CUDA.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    The hot calls (mpg_sample_seeds, mpg_manifold_walk, mpg_estimate,
 *    mpg_guide_*) are asynchronous on that stream and never allocate.
 *  - "device" pointers must be CUDA device (or managed) memory of the current
 *    device; "host" pointers are ordinary host memory.  The caller owns every
 *    query/output buffer; scene and guide objects own deep copies of what is
 *    passed at creation/upload.
 *  - float4 arrays are 16-byte aligned [n][4] float arrays.
 *  - A walk index w in [0, n_recv*spp) belongs to receiver w / spp; its Philox
 *    counter is (walk_id_base + w) (reading R2), so results do not depend on
 *    launch shape, batching or device.
 */
#ifndef MPG_H
#define MPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpg_scene mpg_scene; /* opaque: surfaces + lights + BVH on the device */
typedef struct mpg_guide mpg_guide; /* opaque: guide histogram + sampling tables     */

typedef enum {
    MPG_OK = 0,
    MPG_ERR_INVALID_ARG = 1,
    MPG_ERR_CUDA = 2,
    MPG_ERR_OOM = 3,
    MPG_ERR_UNSUPPORTED = 4,
    MPG_ERR_STATE = 5
} mpg_status;

enum { MPG_SURF_SPHERE = 0, MPG_SURF_QUAD = 1, MPG_SURF_MESH = 2 };
enum { MPG_MAT_CONDUCTOR = 0, MPG_MAT_DIELECTRIC = 1, MPG_MAT_DIFFUSE = 2 };
enum { MPG_LIGHT_POINT = 0, MPG_LIGHT_QUAD = 1 };
/* seed distributions p(x_S | x_D, x_L) */
enum {
    MPG_SEED_CAP = 0,      /* x_1 uniform by area on the cap of sphere surf_id visible from x_D (init) */
    MPG_SEED_TRIANGLE = 1, /* x_1 uniform in a triangle drawn uniformly among front-facing ones of mesh surf_id */
    MPG_SEED_GUIDE_UV = 2, /* x_1 target from the guide histogram over surface (u,v), defensive alpha=1/2 (Eq. 13) */
    MPG_SEED_GUIDE_DIR = 3, /* configs[4]: n ~ 1/2 P_0 + 1/2 P_e (Eqs. 10, 13); (w_D, tau) by one-sample MIS of the
                              initializer (w_D uniform on the hemisphere, tau traced) and the learned
                              P_e(tau|n) x direction histogram (Eqs. 8, 11); sampler.k = max chain length (<= 6) */
    MPG_SEED_GUIDE_STREE = 4 /* the paper's own guide: as GUIDE_DIR, but P_e(n),
                              P_e(tau|n) come from the STree leaf of (x_D, x_L) and w_D from that leaf's vMF
                              mixture of type tau (Eq. 12); needs a guide from mpg_guide_create_stree */
};
/* per-walk status; "converged" = CONVERGED or OCCLUDED */
enum {
    MPG_WALK_CONVERGED = 0,  /* admissible, sides valid, visible                  */
    MPG_WALK_MAXITER = 1,    /* Newton iteration cap reached                      */
    MPG_WALK_SEED_FAIL = 2,  /* no seed, deduction missed, TIR or type mismatch   */
    MPG_WALK_BAD_SIDE = 3,   /* spurious constraint zero (R8)                     */
    MPG_WALK_DEGENERATE = 4, /* singular block, zero-length segment or NaN        */
    MPG_WALK_OCCLUDED = 5,   /* admissible but V = 0                      */
    MPG_WALK_INACTIVE = 6    /* selective activation (MPG_FLAG_SELECTIVE, R36): the STree
                                leaf of (x_D, x_L) holds no own (non-copy) sample, so specular chain
                                sampling is not activated; the caller path-traces instead.  w = 0 */
};

/* One specular (or diffuse occluder) surface.  Outward normal (R9):
 * sphere: (p-c)/r; quad: normalize(edge_u x edge_v); mesh: (v1-v0)x(v2-v0).
 * eta_in is the medium behind the outward normal, eta_out in front of it.
 * Mesh arrays are HOST pointers, copied at mpg_scene_create. */
typedef struct {
    int32_t kind, mat;
    float eta_in, eta_out, reflectance;
    float center[3], radius;                  /* sphere */
    float origin[3], edge_u[3], edge_v[3];    /* quad: origin + a*edge_u + b*edge_v, a,b in [0,1] */
    const float *positions;                   /* mesh: host [n_vertices*3] */
    const float *normals;                     /* mesh: host [n_vertices*3] shading normals (outward) */
    const int32_t *indices;                   /* mesh: host [n_triangles*3] */
    int32_t n_vertices, n_triangles;
    float roughness;                          /* GGX alpha of a glossy specular surface (0: pure specular).
                                                 Glossy chains (R37): each walk draws one offset
                                                 normal per chain vertex from D(m) cos(theta_m) (Philox
                                                 purpose 11 + i/2, trial 0; reused by all trials) and the
                                                 chain satisfies h || m in the shading frame.  < 0 ->
                                                 MPG_ERR_INVALID_ARG */
} mpg_surface_desc;

/* Emitter (R15): point (intensity emit) or one-sided parallelogram
 * centred at position, emitting along normalize(edge_u x edge_v) (radiance emit). */
typedef struct {
    int32_t kind;
    float emit;
    float position[3], edge_u[3], edge_v[3];
} mpg_light_desc;

/* Chain type and seed distribution.  tau bit i = 1 <=> vertex i+1 refracts (T),
 * else reflects (R) (Eq. 6).  1 <= k <= MPG_KMAX. */
#define MPG_KMAX 8
typedef struct {
    int32_t mode;    /* MPG_SEED_* */
    int32_t surf_id; /* sphere (CAP) or mesh (TRIANGLE) the first vertex is drawn on */
    int32_t k;
    uint32_t tau;
} mpg_sampler_desc;

/* Guide layout (R20): a grid of cells_x*cells_y spatial cells over the receiver
 * plane (x,z) in [grid_origin, grid_origin+grid_extent), each holding bins_x*bins_y
 * bins over the surface parameter (u,v) in [0,1)^2, where the seed target of bin
 * (u,v) is (uv_origin[0]+u*uv_scale[0], uv_plane_y, uv_origin[1]+v*uv_scale[1]). */
typedef struct {
    float grid_origin[2], grid_extent[2];
    int32_t cells_x, cells_y, bins_x, bins_y;
    float uv_origin[2], uv_scale[2], uv_plane_y;
    int32_t domain;  /* 0: bins over surface (u,v) (MPG_SEED_GUIDE_UV); 1: typed direction bins
                        (MPG_SEED_GUIDE_DIR): 126 chain types (n <= 6) x equal-area hemisphere bins
                        u = cos(theta) about +y (bins_x), v = (phi + pi)/(2 pi) (bins_y) */
    int32_t n_types; /* 1 (domain 0) or 126 (domain 1) */
} mpg_guide_desc;

/* flag bits 1 and 2 are reserved (a wavefront variant of round 1, removed: slower on every
   config); any bit other than the two below -> MPG_ERR_INVALID_ARG */
#define MPG_FLAG_NEWTON_F64 4u /* Jacobian blocks, frames and steps in fp64 (default fp32; positions and
                                  the residual are always fp64, R24) */
#define MPG_FLAG_SORT 8u      /* persistent kernel: process the primaries in the order of a key built from
                                  (receiver cell, seed direction) for ray coherence; every walk's result is
                                  unchanged (it depends only on its own walk id) */
#define MPG_FLAG_SELECTIVE 16u /* selective activation (R36), MPG_SEED_GUIDE_STREE only (ignored
                                  otherwise): mpg_sample_seeds marks a walk whose STree leaf has no own
                                  sample (bin = -3) and mpg_manifold_walk returns MPG_WALK_INACTIVE for it
                                  (the rendering stage's switch to path tracing) */

typedef struct {
    int32_t max_iters;     /* Newton cap (BASELINE configs: 20, or 40 for k=6)       */
    float tol;             /* ||C||_inf threshold (1e-5)                              */
    float beta0;           /* initial step scale (1)                                  */
    int32_t trials;        /* 1: reciprocal-probability trials (Eq. 15); 0: walk only */
    uint32_t k_max;        /* trial cap (1024); truncation counted                    */
    float same_chain_eps;  /* 0 => 1e-4 * scene extent (R17/SPEC.md:280)              */
    float ray_eps;         /* 0 => 1e-4 * scene extent (R10)                          */
    uint32_t flags;        /* MPG_FLAG_* (0 = default persistent kernel)              */
    uint64_t seed;         /* Philox key                                              */
    uint64_t walk_id_base; /* added to the walk index in the Philox counter          */
    int32_t max_iters_long;/* Newton cap for chains with k >= 3 (0: max_iters)        */
    int32_t recip_repeats; /* M >= 2: the reciprocal probability is estimated M times and averaged
                              (R x M / TR x M, Fig. "repber"): repetition r runs its trials
                              with Philox trial counter r*2^20 + t; trials[w] = sum of the M counts,
                              w = T * (sum/M) / (P(n) pdf_L).  0 or 1: one estimate.  Needs k_max < 2^20;
                              repetitions r >= 1 run only the trials of walks that converged; stats:
                              walks, converged,
                              primary_iters and by_status count one pass, work counters all passes */
} mpg_walk_opts;

/* Configurations (x_D, x_L): receivers; walk w uses receiver w / spp. */
typedef struct {
    const float *xD; /* device float4 [n_recv] (xyz used) */
    const float *nD; /* device float4 [n_recv] receiver normals */
    int64_t n_recv;
    int32_t spp;     /* walks per receiver, >= 1 */
} mpg_query;

/* Seeds (mpg_sample_seeds output, mpg_manifold_walk input); device, length n. */
typedef struct {
    float *xL;       /* float4 [n]: light sample x_L, w = its pdf (area x choice)     */
    float *target;   /* float4 [n]: deduction target (ray x_D -> target gives x_1)   */
    int32_t *bin;    /* [n]: drawn bin (GUIDE_UV/DIR) or triangle (TRIANGLE); -1 none, -2 seed failure */
    uint32_t *ctype; /* [n]: chain length n (bits 0-3) | tau or initializer bits (4-11) | learned (12) */
    float *pn;       /* [n]: P(n) of the length mixture (1 for fixed-length samplers) */
} mpg_seed_buf;

/* Walk outputs; device, length n (chain: kmax planes of n float4). */
typedef struct {
    float *chain;      /* float4 [k][n]: vertex i of walk w at chain[(i*n + w)*4]; w = prim id bits (int; -1 analytic) */
    uint8_t *status;   /* [n] MPG_WALK_* of the primary walk                     */
    uint16_t *iters;   /* [n] Newton iterations of the primary walk              */
    float *G;          /* [n] generalized geometric term incl. V         */
    float *T;          /* [n] throughput kappa*G*L_o (Eq. 2)                     */
    float *w;          /* [n] weight T*<1/P>/pdf_L (Eqs. 9, 15); 0 if no chain   */
    uint32_t *trials;  /* [n] geometric trial count k (0 if not run)             */
    uint16_t *ctype;   /* [n] primary chain type: n (bits 0-3) | tau << 4 (bit i: vertex i+1 is T) */
} mpg_walk_buf;

typedef struct {
    unsigned long long walks;         /* primary walks processed                     */
    unsigned long long converged;     /* CONVERGED or OCCLUDED primaries             */
    unsigned long long newton_iters;  /* all Newton iterations incl. trials          */
    unsigned long long primary_iters; /* Newton iterations of primaries              */
    unsigned long long attempts;      /* seed draws incl. trials                     */
    unsigned long long rays;          /* closest-hit + any-hit rays                  */
    unsigned long long trials;        /* sum of k over walks that ran trials         */
    unsigned long long truncated;     /* trial loops that hit k_max                  */
    unsigned long long node_visits;   /* BVH inner nodes visited                     */
    unsigned long long tri_tests;     /* ray-triangle tests                          */
    unsigned long long vertex_iters;  /* sum over Newton iterations of k (solves)    */
    unsigned long long by_status[8];
} mpg_walk_stats;

typedef struct {
    float extent;      /* bbox diagonal of surfaces + lights (R10) */
    int32_t n_surf, n_light, n_tri, n_nodes;
    int32_t bvh_width; /* 2 (binary nodes) or 4 (collapsed 4-wide nodes) */
    size_t device_bytes;
} mpg_scene_info;

/* Build the device scene: copies all descriptors and mesh arrays (host), builds
 * a binned-SAH BVH over all mesh triangles (host, C++), uploads it.  Synchronous.
 * The binary tree is collapsed to 4-wide nodes for scenes of >= 65,536
 * triangles (environment MPG_BVH_WIDTH=2|4 overrides); traversal results are
 * identical, only the node visits differ. */
mpg_status mpg_scene_create(const mpg_surface_desc *surfaces, int32_t n_surf, const mpg_light_desc *lights,
                            int32_t n_light, void *stream, mpg_scene **out);
mpg_status mpg_scene_destroy(mpg_scene *scene);
mpg_status mpg_scene_get_info(const mpg_scene *scene, mpg_scene_info *info);

/* ---- STree + vMF guide (§5.5-5.6; R28-R31) ----
 * One sub-path sample of an iteration (Eq. 9): its configuration (x_D, x_L), the
 * solved direction w_D* = normalize(x_1* - x_D), its weight w = T <1/P> and its
 * chain type 2^n - 2 + tau (n <= 6).  A record is a sample iff w > 0 and
 * 0 <= type < 126.  48 bytes, device arrays. */
typedef struct {
    float xD[3], xL[3], omega[3], w;
    int32_t type, pad;
} mpg_guide_sample;

typedef struct {
    int64_t max_samples;  /* record capacity between two rebuilds (all ranks' records for exchanges) */
    float eps;            /* overlap fraction of the split (0.1, P:523 footnote)           */
    float c_thr;          /* leaf threshold c sqrt|S| (1)                           */
    float kappa_min;      /* vMF concentration kappa_i = sigma_i'^-2 (Eq. 12) is   */
    float kappa_max;      /* clamped to [kappa_min, kappa_max]; the paper's Eq. 12 is 0 /
                             FLT_MAX (no clamp; sigma' = 0 -> kappa_max; a lone lobe -> 1, R30).
                             [1, 300] is the measured product option (R30b: fewer fireflies
                             on configs[4] than 3e3 / 1e4 / unclamped).  kappa_min < 0 or
                             kappa_max < kappa_min -> MPG_ERR_INVALID_ARG                  */
    int32_t max_depth;    /* 32                                                            */
    int32_t keep_all;     /* 0: fit from the last iteration's samples only (the paper's default,
                             P:426 footnote, records cleared by each rebuild); 1: from all samples
                             encountered so far (the footnote's alternative, Reibold et al.), records
                             kept until max_samples */
} mpg_stree_desc;

/* counts of the current tree: n_nodes, n_leaves, root_ref (>= 0 node, < 0 ~leaf),
 * thr, n_valid (samples it was built from), n_lobes */
typedef struct {
    int64_t n_nodes, n_leaves, root_ref, thr, n_valid, n_lobes;
} mpg_stree_info;

/* Create an STree + vMF guide: empty tree (learned branch absent, like mpg_guide_reset). */
mpg_status mpg_guide_create_stree(const mpg_stree_desc *desc, mpg_guide **out);
/* Append the n = n_recv*spp walks of one call as sample records (x_L from seeds->xL, w_D* from
 * walks->chain vertex 0, type from walks->ctype, w from walks->w; records of walks that are
 * not samples get w = 0).  Asynchronous.  MPG_ERR_INVALID_ARG past max_samples. */
mpg_status mpg_guide_record_samples(mpg_guide *guide, const mpg_query *query, const mpg_seed_buf *seeds,
                                    const mpg_walk_buf *walks, int64_t n, void *stream);
/* Glossy separator (Eq. 14; R35): subsequent mpg_guide_record_samples
 * weight every sample by the separator BSDF, a GGX(alpha) microfacet lobe
 * rho = D(h) / (4 cos_v cos_D) with h = normalize(w_v + w_D*): wv = device float4 [n_recv] unit
 * directions from x_D towards the viewer, nD = the receivers' normals (float4 [n_recv]); the
 * caller keeps both alive.  wv = nD = NULL: diffuse separator (weights unchanged). */
mpg_status mpg_guide_set_separator(mpg_guide *guide, const float *wv, const float *nD, float alpha);
/* Replace the recorded samples by n device records (multi-process exchange, tests). */
mpg_status mpg_guide_set_samples(mpg_guide *guide, const mpg_guide_sample *records, int64_t n, void *stream);
/* Copy the recorded samples to device `records` (capacity >= *n on entry; *n = count on return). */
mpg_status mpg_guide_get_samples(const mpg_guide *guide, mpg_guide_sample *records, int64_t *n, void *stream);
/* For an STree guide, mpg_guide_rebuild builds the tree and the per-leaf tables on the GPU
 * from the recorded samples ("last iteration only", P:426 footnote) and clears them; it
 * synchronizes `stream` once per tree level.  mpg_guide_reset empties the tree. */
mpg_status mpg_guide_stree_info(const mpg_guide *guide, mpg_stree_info *info);
/* Device copies of the tree for tests (sizes from mpg_guide_stree_info; any may be NULL):
 * nodes int4 [n_nodes] (split bits, axis, child0, child1; child < 0 = ~leaf), leaf_begin /
 * leaf_count int64 [n_leaves] into leaf_ids int32 [n_lobes] (record indices, leaf order),
 * grp_off int32 [n_leaves][127], lobe_sample int32 [n_lobes], lobe_prefix u64 [n_lobes],
 * lobe_mu float4 [n_lobes] (mu, kappa), n_prefix u64 [n_leaves][6], type_prefix u64 [n_leaves][126],
 * leaf_own int32 [n_leaves]: samples whose own key descends to the leaf, i.e. the leaf's samples
 * without the overlap copies (selective activation, R36). */
mpg_status mpg_guide_download_stree(const mpg_guide *guide, int32_t *nodes, int64_t *leaf_begin, int64_t *leaf_count,
                                    int32_t *leaf_ids, int32_t *grp_off, int32_t *lobe_sample, uint64_t *lobe_prefix,
                                    float *lobe_mu, uint64_t *n_prefix, uint64_t *type_prefix, int32_t *leaf_own,
                                    void *stream);

/* ---- photon-based initial distribution (R33) ----
 * Trace n_photons photons from the emitters (uniform light choice, cosine-weighted area
 * lights, isotropic point lights; power n_lights * Phi / n_photons) through the specular
 * surfaces (R with probability F at dielectrics, conductors R with weight rho; diffuse
 * surfaces absorb) until they cross the receiver plane against its normal.  records
 * (device, n_photons) gets one mpg_guide_sample per photon: landed after 1..max_vertices
 * specular vertices -> (x_D, x_L, w_D*, type, w = power), else w = 0, type = -1.  Feed them
 * to an STree guide (mpg_guide_set_samples + mpg_guide_rebuild) as the initial guide.
 * Philox counters (photon_id_base + p, purpose 8 / 9 / 10, trial). Asynchronous. */
typedef struct {
    int64_t n_photons;
    uint64_t seed, photon_id_base;
    float plane_point[3], plane_normal[3];
    int32_t max_vertices;  /* 1..6 */
    float ray_eps;         /* 0 => 1e-4 * scene extent */
} mpg_photon_desc;
mpg_status mpg_trace_photons(const mpg_scene *scene, const mpg_photon_desc *desc, mpg_guide_sample *records,
                             void *stream);

/* Debug/test entry: closest specular (spec_only=1) or any-surface hit of n rays.
 * orig/dir: device float4 [n]; outputs device: t [n], prim [n] (original triangle id or -1),
 * surf [n] (-1 = miss). */
mpg_status mpg_trace_rays(const mpg_scene *scene, const float *orig, const float *dir, int64_t n, float tmin,
                          int32_t spec_only, float *t, int32_t *prim, int32_t *surf, void *stream);

/* Guide (BASELINE.json histogram stand-in for P:424-482, R20). */
mpg_status mpg_guide_create(const mpg_guide_desc *desc, mpg_guide **out);
mpg_status mpg_guide_destroy(mpg_guide *guide);
/* energies: device [cells][n_types][bins] float >= 0; builds the integer sampling tables (R20/R22). */
mpg_status mpg_guide_upload(mpg_guide *guide, const float *energy, void *stream);
/* learned branch absent: uniform tables, histogram zeroed. */
mpg_status mpg_guide_reset(mpg_guide *guide, void *stream);
/* histogram[cell(x_D)][bin(x_1*)] += w for walks with status CONVERGED and w > 0 (Eq. 9). */
mpg_status mpg_guide_accumulate(mpg_guide *guide, const mpg_query *query, const mpg_walk_buf *walks, int64_t n,
                                void *stream);
/* tables <- histogram ("last iteration only", P:426 footnote); histogram zeroed. */
mpg_status mpg_guide_rebuild(mpg_guide *guide, void *stream);
/* copies: histogram -> energy (device [cells][n_types][bins] float); tables -> prefix (domain 0:
 * device [cells][bins] u64).  Either may be NULL. */
mpg_status mpg_guide_download(const mpg_guide *guide, float *energy, uint64_t *prefix, void *stream);
/* Overwrite the accumulation histogram with `energy` (device [cells][n_types][bins] float), leaving
 * the sampling tables untouched: the exchange step of a multi-process progressive loop
 * -- accumulate -> download -> all-reduce(sum) over ranks -> set_histogram ->
 * rebuild, so every rank fits the next guide from the samples of all ranks (the
 * samples of the last iteration).  Asynchronous on `stream`; energy must not alias it. */
mpg_status mpg_guide_set_histogram(mpg_guide *guide, const float *energy, void *stream);
/* domain 1 tables: n_prefix [cells][6] u64, type_prefix [cells][126] u64, dir_prefix [cells][126][bins] u32. */
mpg_status mpg_guide_download_dir_tables(const mpg_guide *guide, uint64_t *n_prefix, uint64_t *type_prefix,
                                         uint32_t *dir_prefix, void *stream);

/* Light samples + seed targets for the n = n_recv*spp primary walks (trial 0). */
mpg_status mpg_sample_seeds(const mpg_scene *scene, const mpg_guide *guide, const mpg_sampler_desc *sampler,
                            const mpg_query *query, const mpg_walk_opts *opts, mpg_seed_buf *seeds, void *stream);

/* Workspace bytes mpg_manifold_walk needs for n walks of chain length sampler->k
 * (coherence-sort keys and permutation, trial entries/items, R x M buffers). */
size_t mpg_walk_workspace_size(int64_t n, const mpg_sampler_desc *sampler, const mpg_walk_opts *opts);

/* The batched manifold walk: per walk, deduce the seed chain
 * (Eq. 6), Newton-iterate the half-vector constraints with ray-traced
 * reprojection, validate sides and visibility, evaluate kappa, G, T (Eq. 2),
 * then (opts->trials) count reciprocal-probability trials k (Eq. 15) and write
 * w = T*k/pdf_L.  stats (device, may be NULL) is overwritten. */
mpg_status mpg_manifold_walk(const mpg_scene *scene, const mpg_guide *guide, const mpg_sampler_desc *sampler,
                             const mpg_query *query, const mpg_seed_buf *seeds, const mpg_walk_opts *opts,
                             mpg_walk_buf *out, mpg_walk_stats *stats, void *workspace, size_t workspace_bytes,
                             void *stream);

/* Estimator (Eq. 3): mean[r] = (1/spp) sum_s w[r*spp+s]; var (nullable) = sample variance. */
mpg_status mpg_estimate(const float *w, int64_t n_recv, int32_t spp, float *mean, float *var, void *stream);

/* Render-pass splat (Eq. 3 across passes, "never splat the samples
 * produced in the training stage"): sum[r] += mean_j w[r*spp+j] and (nullable) sumsq[r] += its
 * square, fp64 device arrays [n_recv] the caller zeroes; image = sum / passes. */
mpg_status mpg_splat(const float *w, int64_t n_recv, int32_t spp, double *sum, double *sumsq, void *stream);

/* Debug: for the next mpg_manifold_walk calls, record (||C||_inf, beta) of every
 * primary Newton iteration of walks w < n_walks into buf[w*stride + 2*it + {0,1}]
 * (device float); buf = NULL disables.  Not thread-safe; for tests and tools. */
mpg_status mpg_debug_trace(float *buf, int64_t n_walks, int32_t stride);

const char *mpg_last_error(void);
int32_t mpg_version(void);
/* Number of kernel launches this library has enqueued since load (host-side
 * counter, all threads; library launches such as cub's radix-sort passes are counted too). */
uint64_t mpg_kernel_launches(void);
/* The paper's online training schedule (R34), host logic of the
 * progressive train/render loop, in passes of one walk per receiver: the training budget
 * is T = floor(train_frac * budget_passes) (0.3); training iterations of 1, 2, 4, ...
 * passes (doubling); after an iteration a new round starts only while less than
 * T/2 is used, otherwise the current iteration continues to T; the remaining
 * budget_passes - T passes render with the final guide and only they are splatted.
 * iters (host, max_iters entries) receives the passes of each training iteration, n_iters
 * their number, render_passes the rest.  Synchronous, no device work.  A budget < 0,
 * train_frac outside [0, 1], NULL outputs or too short an iters array -> MPG_ERR_INVALID_ARG. */
mpg_status mpg_training_schedule(int64_t budget_passes, double train_frac, int64_t *iters, int32_t max_iters,
                                 int32_t *n_iters, int64_t *render_passes);
/* Measurement helper, not on the walk path: FP32 FFMA throughput of the current
 * device in TFLOP/s (8 independent FFMA chains per thread, SMs x 4 blocks of 256
 * threads, `iters` x 128 FFMA per thread, best of `reps` timed launches after one
 * warm-up; CUDA events on `stream`, synchronizes).  The roofline denominator of
 * bench.py.  iters/reps <= 0 or tflops NULL -> MPG_ERR_INVALID_ARG. */
mpg_status mpg_measure_fp32_peak(int32_t iters, int32_t reps, double *tflops, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MPG_H */
