// walk.cuh -- the persistent manifold-walk kernel (sm_100a).
//
// One chain per lane.  Lanes run a small state machine
//   FETCH -> SEED -> DEDUCE(trace k rays) -> SOLVE -> REPROJ(trace k rays) -> SOLVE ... -> END
// at Newton-iteration granularity, so a lane whose walk (or trial) ends takes
// the next work item from a global queue (warp-aggregated atomicAdd) while the
// other lanes of its warp keep iterating: warp execution stays full despite
// iteration counts of 0..max_iters and geometric trial counts (SURVEY §7
// "Divergence").  Deduction and reprojection share one trace loop.
//
// Method: Newton on the stacked generalized-half-vector
// constraints C_i = (s.h, t.h) (R1-R3) with the block-tridiagonal Jacobian
// solved by block Thomas elimination fused with the block evaluation (only
// D'^-1_i, U_i, r'_i survive per vertex), step on the geometric tangent planes
// (R4), sequential ray-traced reprojection with step halving (R5, R6),
// convergence on ||C||_inf < tol (R7), sides (R8), visibility, kappa (R12),
// analytic GGT by one more back-substitution with the 2-column light RHS (R11),
// and reciprocal-probability trials (Eq. 15, R13).
#pragma once
// Occupancy (blocks of 128 per SM the register budget must allow), measured
// (k_walk ms): k <= 2: 6 blocks (80 regs) 41.5 / 8 (64) 39.8 / 10 (48) 39.8 /
// 12 (40) 46.1 on configs[1], 312 / 309 / 334 / 366 on [2] -> 8.  k = 6: 2
// blocks (200+ regs) / 4 (128) / 6 (80) / 8 (64): configs[3] 232 / 170 / 163 /
// 180 ms, but the mixed-length loop of configs[4] 256 / 264 / 279 / 292 ms per
// step -> two instantiations, chosen by the sampler (MINB below).
// (re-measured with the batched attempt boundaries of round 2: 6 / 7 / 8 blocks: configs[2] 226.4 /
// 224.3 / 225.3 ms, configs[1] 42.8 / 42.0 / 42.7 -> 7 blocks, 72 registers)
#ifndef MPG_WALK_MINB2
#define MPG_WALK_MINB2 7
#endif
#ifndef MPG_WALK_MINB_LONG
#define MPG_WALK_MINB_LONG 6   // fixed long chains (configs[3])
#endif
#ifndef MPG_WALK_MINB_MIXED
// per-sample chain length (configs[4]); round 1 (per-lane rays): 2/3/4 blocks 261/255/271 ms;
// round 2 (compacted trace rounds, CMP): 2/3/4/5/6 blocks 269/225/219/235/252 ms
#define MPG_WALK_MINB_MIXED 4
#endif
// MPG_COMPACT: block-synchronous passes whose chain rays are traced in compacted
// rounds -- every lane that needs a ray writes it to a shared-memory slot, the
// block's threads trace the slots in order (full warps), and the lanes read their
// hits back -- instead of each lane tracing its own ray inside its warp
#ifndef MPG_COMPACT
#define MPG_COMPACT 1
#endif
// MPG_TRACE_P = 1: the traversal also forms the fp32 hit point of a triangle hit (A/B knob; 0: three
// loads per chain ray less, the walk refines the hit in fp64 from the vertices anyway)
#ifndef MPG_TRACE_P
#define MPG_TRACE_P 0
#endif
#ifndef MPG_SVC_ALL
#define MPG_SVC_ALL 0   // A/B: batched attempt boundaries in every k_walk instantiation (default: k <= 2 only)
#endif
#include "device_common.cuh"
#include "seed.cuh"
#include "newton.cuh"

enum { PH_FETCH = 0, PH_SEED = 1, PH_DEDUCE = 2, PH_SOLVE = 3, PH_REPROJ = 4, PH_END = 5, PH_IDLE = 6, PH_WAIT = 7,
       PH_VIS = 8 };
#define HARD_NONE 0xffffffffu
enum { ST_CONVERGED = 0, ST_MAXITER = 1, ST_SEED_FAIL = 2, ST_BAD_SIDE = 3, ST_DEGENERATE = 4, ST_OCCLUDED = 5,
       ST_INACTIVE = 6 };

struct TrialHdr {
    unsigned long long queue;   // next primary walk
    unsigned int n_entries;     // hard entries published
    unsigned int item_head;     // next ticket
    unsigned int item_tail;     // items reserved
    unsigned int resolved;      // walks whose output (trials, w) is final
};
#define ITEM_EMPTY 0xffffffffffffffffull

struct WalkParams {
    const float4 *xD, *nD;
    int64_t n_recv, n;
    int spp;
    const float4 *seed_xL, *seed_tgt;
    const int *seed_bin;
    const uint32_t *perm;       // processing order of the primaries (MPG_FLAG_SORT), NULL = walk order
    const uint32_t *seed_ctype; // n | bits << 4 | learned << 12 (may be NULL: fixed type)
    const float *seed_pn;       // P(n) (may be NULL: 1)
    uint16_t *out_ctype;        // primary chain type n | tau << 4 (may be NULL)
    int max_iters_long;
    float4 *chain;
    uint8_t *status;
    uint16_t *iters;
    float *G, *T, *w;
    uint32_t *trials;
    unsigned long long *stats; // mpg_walk_stats as u64[21]
    int max_iters, trials_on;
    uint32_t k_max;
    float tol, beta0, same_eps, ray_eps;
    uint64_t walk_id_base;
    float *dbg;      // debug: [n_dbg][stride] (||C||_inf, beta) per primary iteration, or NULL
    int64_t n_dbg;
    int dbg_stride;
    // Reciprocal-probability trials (Eq. 15) beyond the first `local_trials`
    // (sequential in the lane) make the walk a "hard entry" whose trials run as
    // items (entry e, trial t) in doubling batches; lanes whose primary queue is
    // exhausted take items by ticket from a ring, in the same launch.  k = the
    // smallest successful trial: every trial below it has run (batch order).
    uint32_t trial_base;        // Philox trial counter offset of trials t >= 1 (recip_repeats)
    uint32_t *psurf_out;        // recip_repeats: primary surface ids per walk (written by repetition 0)
    int trials_only;            // recip_repeats r >= 1: primaries are final (outputs of repetition 0); run trials only
    size_t trav_bytes;          // host side: bytes of nodes + triangle positions (L2 window)
    uint32_t local_trials;
    uint32_t item_b0;           // first item batch of a hard entry
    uint32_t item_grow;         // later batches: previous << item_grow
    // ... or previous << item_grow_idle while the unclaimed item backlog is below
    // idle_backlog (most lanes idle in the tail: a larger batch then costs no
    // throughput and saves rounds of trial-walk latency on the critical path)
    uint32_t item_grow_idle, idle_backlog, item_b0_idle;
    uint32_t svc_min, svc_wait; // attempt boundaries served in batches (k_walk): waiting lanes / passes that trigger a service
    uint32_t backoff_max;       // ns, cap of the waiting warps' sleep
    uint32_t hard_cap;          // entries
    uint32_t item_cap;          // item ring capacity (a full ring -> sequential fallback)
    struct TrialHdr *th;        // counters (zeroed before the launch)
    int64_t *e_walk;
    uint32_t *e_psurf, *e_pct, *e_best, *e_pending, *e_issued, *e_batch;
    unsigned long long *items;  // (e << 32 | t); ~0 = not yet written (ring memset to 0xff)
};

// stats slots (mirror mpg_walk_stats field order)
enum { SS_WALKS = 0, SS_CONV, SS_NEWTON, SS_PRIM_IT, SS_ATTEMPTS, SS_RAYS, SS_TRIALS, SS_TRUNC, SS_NODES, SS_TRIS,
       SS_VTX, SS_STATUS0, SS_N = SS_STATUS0 + 8 };

// reflect / refract the propagation direction d at a vertex (deduction, Eq. 6);
// media from the side of d w.r.t. the geometric normal (R9, R14).  Everything in
// fp64 at the fp64 vertex, normals included (an fp32 shading normal at the
// fp32-rounded point tilted the deduced chain by ~1e-7 relative, which the long
// halving sequences of configs[3] amplified into different outcomes, measured):
// the deduced seed chain matches the oracle's to fp64 rounding.
template <bool GL>
__device__ __forceinline__ bool scatter_dir(const DScene &S, double3 &dd, int prim, int surf, double3 p, bool isT,
                                            uint64_t seed, uint64_t wid, int vi) {
    const DSurf &f = S.surf[surf];
    const V3<double> ng = geo_normalR<double>(S, prim, surf, p);
    V3<double> dna, dnb;
    const V3<double> z0 = mk3<double>(0.0, 0.0, 0.0);
    V3<double> nf = shadingR<double>(S, prim, surf, p, z0, z0, dna, dnb);
    if (GL && f.rough > 0.0f) {  // scatter about the offset normal of vertex vi (R37)
        double oa, ob;
        glossy_slopes(S, surf, seed, wid, vi, oa, ob);
        V3<double> s, t;
        onbR(nf, s, t);
        nf = nrmR(nf + s * oa + t * ob);
    }
    double dx = dd.x, dy = dd.y, dz = dd.z, nx = nf.x, ny = nf.y, nz = nf.z;
    double il = rsqrt(nx * nx + ny * ny + nz * nz);
    nx *= il; ny *= il; nz *= il;
    bool outside = (dx * ng.x + dy * ng.y + dz * ng.z) < 0.0;
    double dn = dx * nx + dy * ny + dz * nz;
    if (dn > 0.0) { nx = -nx; ny = -ny; nz = -nz; dn = -dn; }
    double ci = -dn;
    if (!(ci > 0.0)) return false;
    double rx, ry, rz;
    if (!isT) {
        rx = dx + 2.0 * ci * nx; ry = dy + 2.0 * ci * ny; rz = dz + 2.0 * ci * nz;
    } else {
        if (f.mat != 1) return false;
        double e1 = outside ? f.eta_out : f.eta_in, e2 = outside ? f.eta_in : f.eta_out;
        double eta = e1 / e2;
        double k2 = 1.0 - eta * eta * (1.0 - ci * ci);
        if (k2 < 0.0) return false; // TIR
        double c = eta * ci - sqrt(k2);
        rx = eta * dx + c * nx; ry = eta * dy + c * ny; rz = eta * dz + c * nz;
    }
    double ir = rsqrt(rx * rx + ry * ry + rz * rz);
    dd = make_double3(rx * ir, ry * ir, rz * ir);
    return true;
}

// Hit point of the line o + t*(q - o) with the primitive the fp32 traversal
// found, recomputed in fp64 from the fp32 inputs (exact differences) and
// rounded once: the reprojected vertex is within 1/2 ulp of the exact point,
// so the Newton residual is not floored by reprojection noise (which near
// grazing chains reached ~1e-5 in fp32, measured).
//
// Triangle choice at shared edges (R17): the fp32 watertight traversal may pick
// the neighbour of the triangle the exact (fp64) line crosses when the crossing
// lies within fp32 rounding of their common edge.  The plane of the wrong
// neighbour moves the vertex by ~(distance to the edge) x (dihedral angle)
// ~ 1e-9 x extent, which long chaotic walks (k = 6 slabs, 40 halving
// iterations) amplify to a different outcome.  So the fp64 barycentrics of the
// refined point are checked, and while one is negative the point moves to the
// triangle across that edge (mesh adjacency, <= 2 hops): the primitive is then
// the one the exact line crosses, as in the fp64 oracle.  `prim` is updated.
// pf: the traversal's fp32 hit point, or (pf_bary, triangles only) its barycentrics: the fp32 point
// is only the fallback of a line parallel to the triangle's plane
__device__ __forceinline__ double3 refine_hit(const DScene &S, int &prim, int surf, double3 o, double3 q, float3 pf,
                                              const bool pf_bary = false) {
    double ox = o.x, oy = o.y, oz = o.z;
    double dx = q.x - ox, dy = q.y - oy, dz = q.z - oz;
    double t;
    if (prim >= 0) {
        int cur = prim;
        double3 y0 = d3f(pf);
#pragma unroll 1
        for (int hop = 0; hop < 3; hop++) {
            float3 a = xyz(__ldg(S.tpos + TSTRIDE * cur)), b = xyz(__ldg(S.tpos + TSTRIDE * cur + 1)),
                   c = xyz(__ldg(S.tpos + TSTRIDE * cur + 2));
            double e1x = (double)b.x - a.x, e1y = (double)b.y - a.y, e1z = (double)b.z - a.z;
            double e2x = (double)c.x - a.x, e2y = (double)c.y - a.y, e2z = (double)c.z - a.z;
            double nx = e1y * e2z - e1z * e2y, ny = e1z * e2x - e1x * e2z, nz = e1x * e2y - e1y * e2x;
            double den = dx * nx + dy * ny + dz * nz;
            if (den == 0.0) {
                if (hop == 0 && pf_bary) y0 = d3f(a * pf.x + b * pf.y + c * pf.z);
                break;
            }
            t = (((double)a.x - ox) * nx + ((double)a.y - oy) * ny + ((double)a.z - oz) * nz) / den;
            const double3 y = make_double3(ox + t * dx, oy + t * dy, oz + t * dz);
            if (hop == 0) y0 = y;
            if (!S.tadj) { prim = cur; return y; }
            // unnormalized barycentrics (sign = side of each edge): opposite a, b, c
            double pax = (double)a.x - y.x, pay = (double)a.y - y.y, paz = (double)a.z - y.z;
            double pbx = (double)b.x - y.x, pby = (double)b.y - y.y, pbz = (double)b.z - y.z;
            double pcx = (double)c.x - y.x, pcy = (double)c.y - y.y, pcz = (double)c.z - y.z;
            double wa = (pby * pcz - pbz * pcy) * nx + (pbz * pcx - pbx * pcz) * ny + (pbx * pcy - pby * pcx) * nz;
            double wb = (pcy * paz - pcz * pay) * nx + (pcz * pax - pcx * paz) * ny + (pcx * pay - pcy * pax) * nz;
            double wc = (pay * pbz - paz * pby) * nx + (paz * pbx - pax * pbz) * ny + (pax * pby - pay * pbx) * nz;
            if (wa >= 0.0 && wb >= 0.0 && wc >= 0.0) { prim = cur; return y; }
            const int4 nb = __ldg(S.tadj + cur);
            const int nxt = (wa <= wb && wa <= wc) ? nb.x : (wb <= wc ? nb.y : nb.z);
            if (nxt < 0) break;
            cur = nxt;
        }
        return y0;   // no neighbour contains the crossing: keep the traversal's triangle
    } else {
        const DSurf &f = S.surf[surf];
        if (f.kind == 0) {
            double cx = ox - f.center.x, cy = oy - f.center.y, cz = oz - f.center.z;
            double dd = dx * dx + dy * dy + dz * dz;
            double bb = (cx * dx + cy * dy + cz * dz) / dd;
            double rx = cx - bb * dx, ry = cy - bb * dy, rz = cz - bb * dz;
            double disc = ((double)f.radius * f.radius - (rx * rx + ry * ry + rz * rz)) / dd;
            if (disc < 0.0) return d3f(pf);
            double sq = sqrt(disc);
            // the root nearest to the fp32 hit the traversal selected
            double tf = ((double)pf.x - ox) * dx + ((double)pf.y - oy) * dy + ((double)pf.z - oz) * dz;
            tf /= dd;
            double t0 = -bb - sq, t1 = -bb + sq;
            t = fabs(t0 - tf) <= fabs(t1 - tf) ? t0 : t1;
        } else {
            double nx = f.nq.x, ny = f.nq.y, nz = f.nq.z;
            double den = dx * nx + dy * ny + dz * nz;
            if (den == 0.0) return d3f(pf);
            t = (((double)f.origin.x - ox) * nx + ((double)f.origin.y - oy) * ny + ((double)f.origin.z - oz) * nz) / den;
        }
    }
    return make_double3(ox + t * dx, oy + t * dy, oz + t * dz);
}

// Trace the k chain vertices from x_D: deduction (scatter by tau) or
// reprojection toward q_i (must stay on surf_i).  Rolled loop: one traversal
// site.  y/yp/ys/q live in local memory (dynamic index).
// returns 0 on success, else 1 + (i << 4) | reason (1 miss, 2 wrong surface, 3 zero length, 4 scatter)
// Traversal runs in fp32 (the hit/miss and which-primitive decisions); the hit
// point is recomputed in fp64 on the exact line (refine_hit) and kept in fp64.
// Deduction resolves the type string: vertex i takes bit i of `bits`, except
// that the initializer (learned = false) always reflects on a conductor; T on
// a conductor fails (R22, R14).  The resolved string is returned in tau_res.
enum { TR_REPROJ = 0, TR_DEDUCE = 1, TR_VIS = 2 };
// TR_VIS: the k+1 visibility segments x_D -> x_1 -> ... -> x_k -> x_L of the
// converged chain x (any hit against all surfaces); returns 5 if occluded.
// One traversal call site serves all three modes, so lanes tracing visibility
// traverse together with warp-mates that reproject (no separate low-occupancy
// visibility traversal).
// Reprojection targets q_i = x_i + beta dq_i are formed here from the chain and its
// step (no q array survives between the Newton step and the trace).
template <int KMAX, int W, typename R, bool GL>
__device__ __forceinline__ int trace_chain(const DScene &S, int mode, int k, uint32_t bits, bool learned,
                                           float3 xD, float3 xL, float3 tgt, const V3<R> (&dq)[KMAX], float beta,
                                           const double3 (&x)[KMAX], const int (&hint)[KMAX],
                                           uint32_t surf_req, float eps, double3 (&y)[KMAX], int (&yp)[KMAX],
                                           int (&ys)[KMAX], LaneStats &st, uint32_t &tau_res, unsigned *s_rays,
                                           uint64_t seed, uint64_t wid, const float4 *top = nullptr) {
    const bool deduce = mode == TR_DEDUCE, vis = mode == TR_VIS;
    uint32_t res = 0;
    double3 o = d3f(xD);
    double3 dd = make_double3(0.0, 0.0, 0.0);
    if (deduce) {
        double3 v = d3f(tgt) - o;
        double l2 = ddot(v, v);
        if (!(l2 > 0.0)) return 3;
        dd = v * rsqrt(l2);
    }
    int pprim = -1, psurf = 0;
    const int nr = vis ? k + 1 : k;
#pragma unroll 1
    for (int i = 0; i < nr; i++) {
        float3 of, d;
        float tmax = 3.0e38f;
        if (vis) {
            const float3 a = i == 0 ? xD : f3d(rget(x, i - 1));
            const float3 b = i == k ? xL : f3d(rget(x, i));
            const float3 ab = b - a;
            const float l = len(ab);
            of = a;
            d = ab * (1.0f / l);
            tmax = l - eps;
        } else {
            if (!deduce) {
                double3 v = (rget(x, i) + tod(rget(dq, i)) * (double)beta) - o;
                double l2 = ddot(v, v);
                if (!(l2 > 0.0)) return 3 | (i << 4);
                dd = v * rsqrt(l2);
            } else if (i > 0) {
                if (!scatter_dir<GL>(S, dd, pprim, psurf, o, (res >> (i - 1)) & 1u, seed, wid, i - 1)) return 4 | (i << 4);
            }
            of = f3d(o);
            d = nrmz(f3d(dd));
        }
        // rays are counted with a shared-memory atomic on the lane's own slot: an
        // atomic in this loop makes ptxas emit a YIELD at its head, which lets lanes
        // that are done with ray i go on while warp-mates still traverse (measured
        // k_walk -17 % configs[1], -7 % [2], -13 % [3] against a register counter)
        atomicAdd(s_rays, 1u);
        Hit h;
        const bool hit = trace<W, MPG_TRACE_P != 0>(S, of, d, eps, tmax, !vis, vis, h, st, mode == TR_REPROJ ? rget(hint, i) : -1,
                                                    top);
        if (vis) {
            if (hit) return 5;
            continue;
        }
        if (!hit) return 1 | (i << 4);
        if (!deduce && h.surf != (int)((surf_req >> (4 * i)) & 15u)) return 2 | (i << 4);
        if (deduce) {
            uint32_t bit = (bits >> i) & 1u;
            const int mat = S.surf[h.surf].mat;
            if (!learned && mat == 0) bit = 0u;
            if (bit && mat != 1) return 4 | (i << 4);
            res |= bit << i;
        }
        const double3 yi = refine_hit(S, h.prim, h.surf, o, deduce ? o + dd : rget(x, i) + tod(rget(dq, i)) * (double)beta,
                                      h.p, MPG_TRACE_P == 0);   // may move h.prim across a shared edge
        rset(y, i, yi);
        rset(yp, i, h.prim);
        rset(ys, i, h.surf);
        pprim = h.prim;
        psurf = h.surf;
        o = yi;
    }
    tau_res = res;
    return 0;
}

// ---- reciprocal-probability trial bookkeeping (hard entries / items) ----
// final output of a walk with trial count kk (Eq. 15: w = T k / (P(n) pdf_L),
// P(n) and pdf_L of the primary sample)
__device__ __forceinline__ void trial_finalize(const WalkParams &P, int64_t w, uint32_t kk, bool truncated,
                                               unsigned *s_stats) {
    P.trials[w] = kk;
    const float pn = P.seed_pn ? __ldg(P.seed_pn + w) : 1.0f;
    P.w[w] = __ldcg(P.T + w) * (float)kk / (pn * __ldg(P.seed_xL + w).w);
    atomicAdd(&s_stats[SS_TRIALS], kk);
    if (truncated) atomicAdd(&s_stats[SS_TRUNC], 1u);
}
// walks a lane has made final are counted in a register and published when the
// lane runs out of primaries (PH_WAIT): one atomic per lane, not per walk
#define walk_resolved(P) (my_resolved++)
// publish items (e, t0 .. t0+B-1); false if the ring is full
__device__ __forceinline__ bool items_push(const WalkParams &P, uint32_t e, uint32_t t0, uint32_t B) {
    unsigned base = atomicAdd(&P.th->item_tail, B);
    if ((unsigned long long)base + B > P.item_cap) return false;
    MPG_CHECK((unsigned long long)base + B <= P.item_cap);
    for (uint32_t j = 0; j < B; j++)
        *(volatile unsigned long long *)(P.items + base + j) = ((unsigned long long)e << 32) | (t0 + j);
    return true;
}

// the primary queue is exhausted (this warp saw it, or the global counter says so)
__device__ __forceinline__ bool queue_drained(const WalkParams &P, bool drained) {
    return drained || __ldcg(&P.th->queue) >= (unsigned long long)P.n;
}
// make walk w a hard entry whose trials last+1 .. run as items (first batch
// item_b0); false (and seq_only: the walk's remaining trials stay in this lane,
// it never asks again) if the entry table or the ring is full.  A full table is
// seen with a plain load first, so the 32-bit counter stops growing once it
// reaches hard_cap (no wrap-around onto live entries, no atomic per trial).
__device__ __forceinline__ bool hard_publish(const WalkParams &P, int64_t w, uint32_t psurf, int pk, uint32_t ptau,
                                             uint32_t last, bool &seq_only) {
    if (*(volatile unsigned int *)&P.th->n_entries >= P.hard_cap) { seq_only = true; return false; }
    unsigned int e = atomicAdd(&P.th->n_entries, 1u);
    if (e >= P.hard_cap) { seq_only = true; return false; }
    const unsigned backlog = *(volatile unsigned *)&P.th->item_tail - *(volatile unsigned *)&P.th->item_head;
    const bool idle = (int)backlog < (int)P.idle_backlog && __ldcg(&P.th->queue) >= (unsigned long long)P.n;
    const uint32_t B = min(idle ? P.item_b0_idle : P.item_b0, P.k_max - last);
    MPG_CHECK(e < P.hard_cap && w >= 0 && w < P.n);
    P.e_walk[e] = w;
    P.e_psurf[e] = psurf;
    P.e_pct[e] = (uint32_t)pk | (ptau << 4);
    P.e_best[e] = HARD_NONE;
    P.e_batch[e] = B;
    P.e_pending[e] = B;
    P.e_issued[e] = last + B;
    __threadfence();
    const bool ok = items_push(P, e, last + 1, B);
    if (!ok) seq_only = true;
    return ok;
}

#ifdef MPG_TIMELINE
// diagnostic build only (tools/timeline.py): per 65.5-us bucket of %globaltimer,
// [warp iterations, tracing, working, waiting, primary (trial 0), item lanes]
#define TL_W 6
__device__ unsigned long long g_tl[1024 * TL_W];
__device__ unsigned g_tl_shift = 16;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// the end of a trace: the lane consumes its trace result (deduced / reprojected chain, or
// the visibility of a converged primary)
#define MPG_TRACE_TAIL \
            if (mode == TR_VIS) { \
                occluded = !ok; \
                phase = PH_END; \
            } else { \
            if (ok && ded) tau = tres; \
            if (!ok && !ded && P.dbg && trial == 0 && w < P.n_dbg && 2 * it + 3 < P.dbg_stride) \
                P.dbg[w * P.dbg_stride + 2 * (it + 1)] = -(float)(why + 1); \
            if (ok) { \
_Pragma("unroll") \
                for (int i = 0; i < KMAX; i++) { \
                    if (i >= k) break; \
                    x[i] = y[i]; prim[i] = yp[i]; surf[i] = ys[i]; \
                } \
                fresh = true; \
                if (ded) { beta = P.beta0; it = 0; } \
                else { beta = fminf(1.0f, 2.0f * beta); it++; } \
                phase = PH_SOLVE; \
            } else if (ded) { \
                end_status = ST_SEED_FAIL; \
                phase = PH_END; \
            } else { \
                beta *= 0.5f; \
                it++; \
                phase = PH_SOLVE; \
            } \
            } \

// GL: glossy scenes (offset normals, R37) -- the glossy code is compiled only into the kernels
// for scenes with a rough surface; CMP: compacted trace rounds (MPG_COMPACT above)
template <int KMAX, typename R, int W, int MINB, bool GL, bool CMP>
__global__ void __launch_bounds__(128, MINB) k_walk(const DScene S, const SeedCtx g, const WalkParams P) {
    // ray slots of the compacted trace rounds (CMP): origin + tmax, direction + mode, hint;
    // hits: point, primitive + surface
    constexpr int NS = CMP ? 128 : 1;
    __shared__ float4 s_ro[NS], s_rd[NS], s_hp[NS];
    __shared__ int2 s_hs[NS];
    __shared__ int s_rh[NS];
    __shared__ int s_wcnt[4];
    const int warp = threadIdx.x >> 5;
    // per-block walk counters in 32 bits (native shared atomics; 64-bit shared atomicAdd
    // compiles to a CAS loop): a block makes at most ~2^25 walks final per launch
    __shared__ unsigned s_stats[SS_N];
    __shared__ unsigned s_rays[128];   // chain rays per thread (see trace_chain)
    for (int i = threadIdx.x; i < SS_N; i += blockDim.x) s_stats[i] = 0u;
    s_rays[threadIdx.x] = 0u;
    // the first levels of the BVH (breadth-first at the front of the node array) in shared memory
    constexpr int NTOPF4 = MPG_TOP_NODES > 0 ? MPG_TOP_NODES * NODE_F4(W) : 1;
    __shared__ float4 s_top[NTOPF4];
    const float4 *top = nullptr;
    if (MPG_TOP_NODES > 0 && S.n_nodes >= MPG_TOP_NODES) {
        for (int i = threadIdx.x; i < NTOPF4; i += blockDim.x) s_top[i] = __ldg(S.nodes + i);
        top = s_top;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    // chain type of the current attempt (per lane: configs[4] draws n and tau per sample)
    int k = g.k, pk = g.k;
    uint32_t tau = g.tau, ptau = g.tau;

    // lane state
    int phase = PH_FETCH;
    int64_t w = -1;
    uint32_t trial = 0;
    int end_status = 0;
    float3 xD = f3(0, 0, 0), xL = f3(0, 0, 0);
    float pdfL = 1.f, Tprim = 0.f;
    float Gc = 0.f, Tc = 0.f;   // G, T of a converged primary (computed before its visibility rays)
    int lid = 0;
    int it = 0;
    float beta = 1.f;
    bool fresh = false;
    uint32_t psurf = 0; // primary surf ids, 4 bits each
    // persistent chain state: the vertices, their primitives and the Newton step (kept
    // for step halving); the Jacobian blocks, frames and GGT live only inside the
    // SOLVE block below (transient), so they never stay live across a trace
    double3 x[KMAX];
    V3<R> dq[KMAX];
    int prim[KMAX], surf[KMAX];
    double3 y[KMAX];
    int yp[KMAX], ys[KMAX];
    bool occluded = false;   // visibility of a converged primary (PH_VIS)
#pragma unroll
    for (int i = 0; i < KMAX; i++) {
        x[i] = make_double3(0.0, 0.0, 0.0);
        dq[i] = mk3<R>(0, 0, 0);
        prim[i] = -1; surf[i] = 0;
    }
    LaneStats ls = {0u, 0u, 0u};
    uint32_t c_newton = 0, c_vtx = 0, c_attempts = 0;

    uint32_t my_resolved = 0; // walks made final by this lane, not yet added to th->resolved
    unsigned backoff = 256u;  // ns, while the whole warp waits for trial items
    bool drained = false;     // warp-uniform: this warp saw the primary queue exhausted
    int item_e = -1;          // hard entry of the trial item this lane runs (-1: none)
    long long ticket = -1;    // item-ring ticket while waiting for an item
    bool seq_only = false;    // trials continued in this lane after a full item ring
    // Attempt boundaries in batches (non-compact kernels): the end-of-attempt, fetch and seed sections
    // cost a warp the same whether one lane or ten are in them, and with ~1.7 lanes of a warp ending
    // an attempt per pass they used to run in ~83 % of the passes at 1.5 active lanes (and pull their
    // code through the instruction cache every pass).  A lane whose attempt ended now waits until
    // svc_min lanes of its warp wait, or svc_wait passes (WalkParams), and the warp then serves them
    // together.  A walk's arithmetic does not depend on when it is served: outputs are unchanged.
    bool svc = true;        // warp-uniform: this pass serves the fetch / seed sections (decided at the last end section)
    int svc_since = 0;
    while (true) {
        // ---- fetch a primary walk (warp-aggregated) ------------------------
        unsigned need = __ballot_sync(MPG_FULL, phase == PH_FETCH);
        if (!svc) need = 0u;
        if (need) {
            int leader = __ffs(need) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&P.th->queue, (unsigned long long)__popc(need));
            base = __shfl_sync(MPG_FULL, base, leader);
            if (base + __popc(need) >= (unsigned long long)P.n) drained = true;   // warp-uniform
            if (phase == PH_FETCH) {
                int64_t idx = (int64_t)base + __popc(need & ((1u << lane) - 1u));
                item_e = -1;
                seq_only = false;
                if (idx < P.n) {
                    w = P.perm ? (int64_t)__ldg(P.perm + idx) : idx;
                    trial = 0;
                    const uint32_t rcv = (uint32_t)w / (uint32_t)P.spp;   // n < 2^31 (mpg_manifold_walk): no 64-bit division
                    xD = xyz(__ldg(P.xD + rcv));
                    float4 l4 = __ldg(P.seed_xL + w);
                    xL = xyz(l4);
                    pdfL = l4.w;
                    lid = 0;
                    if (S.n_light > 1) lid = (int)uidx(rng_draw(g.seed, P.walk_id_base + w, 0u, 0u).z, (uint32_t)S.n_light);
                    phase = PH_SEED;
                    if (P.trials_only) {
                        // R x M repetition r >= 1 (R32): the primary chain, its type, surfaces and T
                        // are the outputs of repetition 0; only the trial sequence r*2^20 + t runs
                        const float T0 = P.T[w];
                        if (P.status[w] == ST_CONVERGED && T0 > 0.0f && P.trials_on) {
                            const uint32_t ct = P.out_ctype ? (uint32_t)P.out_ctype[w] : ((uint32_t)g.k | (g.tau << 4));
                            pk = (int)(ct & 15u);
                            ptau = ct >> 4;
                            psurf = P.psurf_out[w];
                            Tprim = T0;
                            trial = 1;
                        } else {
                            P.trials[w] = 0;
                            P.w[w] = 0.0f;
                            walk_resolved(P);
                            phase = PH_FETCH;
                        }
                    }
                } else {
                    phase = PH_WAIT;   // primaries exhausted: trial items
                }
            }
        }
        // ---- take a trial item by ticket, or stop when every walk is final ----
        // (only once the warp has drained the primary queue: no extra warp-wide
        // synchronisation in the main phase)
        if (drained) {
        {   // tickets for lanes without one: one atomic per warp
            unsigned needt = __ballot_sync(MPG_FULL, phase == PH_WAIT && ticket < 0);
            if (needt) {
                int leader = __ffs(needt) - 1;
                unsigned base = 0;
                if (lane == leader) base = atomicAdd(&P.th->item_head, (unsigned)__popc(needt));
                base = __shfl_sync(MPG_FULL, base, leader);
                if (phase == PH_WAIT && ticket < 0) ticket = (long long)(base + __popc(needt & ((1u << lane) - 1u)));
            }
        }
        if (phase == PH_WAIT) {
            if (my_resolved) {
                __threadfence();   // this lane's outputs before the count that ends the launch
                atomicAdd(&P.th->resolved, my_resolved);
                my_resolved = 0;
            }
            unsigned long long wd = ticket >= 0 && ticket < (long long)P.item_cap
                                        ? *(volatile unsigned long long *)(P.items + ticket) : ITEM_EMPTY;
            if (wd != ITEM_EMPTY) {
                ticket = -1;
                item_e = (int)(wd >> 32);
                trial = (uint32_t)wd;
                // entries and primary chains are written by other SMs during this launch:
                // read them through L2 (ld.global.cg), never from a possibly stale L1 line
                MPG_CHECK(item_e >= 0 && (uint32_t)item_e < P.hard_cap);
                w = __ldcg(P.e_walk + item_e);
                MPG_CHECK(w >= 0 && w < P.n);
                psurf = __ldcg(P.e_psurf + item_e);
                uint32_t pct = __ldcg(P.e_pct + item_e);
                pk = (int)(pct & 15u);
                ptau = pct >> 4;
                const uint32_t rcv = (uint32_t)w / (uint32_t)P.spp;
                xD = xyz(__ldg(P.xD + rcv));
                float4 l4 = __ldg(P.seed_xL + w);
                xL = xyz(l4);
                pdfL = l4.w;
                lid = 0;
                if (S.n_light > 1) lid = (int)uidx(rng_draw(g.seed, P.walk_id_base + w, 0u, 0u).z, (uint32_t)S.n_light);
                // a trial above an already found success cannot change k: skip its walk
                if (*(volatile uint32_t *)(P.e_best + item_e) < trial) { end_status = ST_SEED_FAIL; it = 0; phase = PH_END; }
                else phase = PH_SEED;
            } else if (*(volatile unsigned int *)&P.th->resolved >= (unsigned int)P.n) {
                phase = PH_IDLE;
            }
        }
        if constexpr (!CMP) {
        const unsigned wst = __reduce_and_sync(MPG_FULL, (phase == PH_IDLE ? 1u : 0u) |
                                                          (phase == PH_IDLE || phase == PH_WAIT ? 2u : 0u));
        if (wst & 1u) break;
        if (wst & 2u) {
            // the whole warp waits for trial items: back off (polling lanes would
            // otherwise flood L2 while the remaining lanes finish their walks)
            __nanosleep(backoff);
            backoff = min(2u * backoff, P.backoff_max);
            continue;
        }
        backoff = 256u;
        }
        }
        if constexpr (CMP) {
        // block-synchronous passes: the block stops when every lane is idle and backs off
        // while every lane waits for trial items
        if (__syncthreads_and(phase == PH_IDLE)) break;
        if (__syncthreads_and(phase == PH_IDLE || phase == PH_WAIT)) {
            __nanosleep(backoff);
            backoff = min(2u * backoff, P.backoff_max);
            continue;
        }
        backoff = 256u;
        }

        // ---- seed ---------------------------------------------------------
        // (the seed target and the type bits are used by the deduction of the same
        // pass only: not loop-carried)
        float3 tgt = f3(0, 0, 0);
        uint32_t bits = g.tau;
        bool learned = true;
        if (phase == PH_SEED && svc) {
            c_attempts++;
            bool ok;
            bool inactive = false;
            if (trial == 0) {
                const int sb = __ldg(P.seed_bin + w);
                ok = sb >= -1;
                inactive = sb == -3;   // selective activation (R36): left to path tracing
                tgt = xyz(__ldg(P.seed_tgt + w));
                if (P.seed_ctype) {
                    uint32_t ct = __ldg(P.seed_ctype + w);
                    k = (int)(ct & 15u);
                    bits = (ct >> 4) & 255u;
                    learned = (ct >> 12) & 1u;
                }
            } else {
                SeedRes sr;
                ok = seed_target(S, g, P.walk_id_base + w, trial + P.trial_base, xD, xL, sr);
                tgt = sr.tgt;
                k = sr.n;
                bits = sr.bits;
                learned = sr.learned;
            }
            k = max(1, min(k, KMAX));
            it = 0;
            if (ok) phase = PH_DEDUCE;
            else { end_status = inactive ? ST_INACTIVE : ST_SEED_FAIL; phase = PH_END; }
        }

#ifdef MPG_TIMELINE
        {
            const bool wk = phase != PH_WAIT && phase != PH_IDLE;
            const unsigned c[5] = {__ballot_sync(MPG_FULL, phase == PH_DEDUCE || phase == PH_REPROJ || phase == PH_VIS),
                                   __ballot_sync(MPG_FULL, wk), __ballot_sync(MPG_FULL, phase == PH_WAIT),
                                   __ballot_sync(MPG_FULL, wk && trial == 0), __ballot_sync(MPG_FULL, wk && item_e >= 0)};
            if (lane == 0) {
                const unsigned b = (unsigned)(gtimer() >> g_tl_shift) & 1023u;
                atomicAdd(&g_tl[TL_W * b], 1ull);
                for (int j = 0; j < 5; j++) atomicAdd(&g_tl[TL_W * b + 1 + j], (unsigned long long)__popc(c[j]));
            }
        }
#endif
        // ---- trace: deduction (Eq. 6) or reprojection --------------------
        // (the two variants share the tail MPG_TRACE_TAIL; each instantiation sees only its own
        // code: the non-compact one is exactly the round-1 structure, A/B-measured)
        if constexpr (!CMP) {
        if (phase == PH_DEDUCE || phase == PH_REPROJ || phase == PH_VIS) {
            bool ded = phase == PH_DEDUCE;
            uint32_t sreq = 0;
#pragma unroll
            for (int i = 0; i < KMAX; i++) sreq |= (uint32_t)(surf[i] & 15) << (4 * i);
            uint32_t tres = tau;
            const int mode = ded ? TR_DEDUCE : (phase == PH_VIS ? TR_VIS : TR_REPROJ);
            int why = trace_chain<KMAX, W, R, GL>(S, mode, k, bits, learned, xD, xL, tgt, dq, beta, x, prim, sreq,
                                                  P.ray_eps, y, yp, ys, ls, tres, &s_rays[threadIdx.x], g.seed,
                                                  P.walk_id_base + w, top);
            bool ok = why == 0;
            MPG_TRACE_TAIL
        }
        } else {
        const bool tracing = phase == PH_DEDUCE || phase == PH_REPROJ || phase == PH_VIS;
        const int tmode = phase == PH_DEDUCE ? TR_DEDUCE : (phase == PH_VIS ? TR_VIS : TR_REPROJ);
        uint32_t tres = 0;
        // The lane's k (or k+1 visibility) rays are traced in rounds: ray i of every
        // tracing lane of the block goes to a shared slot, the block's first M threads
        // trace the M slots (warps start full), and each lane consumes its hit (the
        // body of trace_chain split at the traversal call).  Same rays, same results.
        int ti = -1, tcode = 0, tpp = -1, tps = 0;
        uint32_t sreq = 0;
        tres = 0;
        double3 to = d3f(xD), tdd = make_double3(0.0, 0.0, 0.0);
        if (tracing) {
            ti = 0;
#pragma unroll
            for (int i = 0; i < KMAX; i++) sreq |= (uint32_t)(surf[i] & 15) << (4 * i);
            if (tmode == TR_DEDUCE) {
                const double3 v = d3f(tgt) - to;
                const double l2 = ddot(v, v);
                if (!(l2 > 0.0)) { tcode = 3; ti = -1; }
                else tdd = v * rsqrt(l2);
            }
        }
        const int tnr = tmode == TR_VIS ? k + 1 : k;
        while (__syncthreads_or(ti >= 0)) {
            // 1. this lane's ray ti (top of the trace_chain loop body)
            bool has = ti >= 0;
            float3 of = f3(0.f, 0.f, 0.f), d = f3(0.f, 0.f, 1.f);
            float tmax = 3.0e38f;
            int hint = -1;
            if (has) {
                if (tmode == TR_VIS) {
                    const float3 a = ti == 0 ? xD : f3d(rget(x, ti - 1));
                    const float3 b = ti == k ? xL : f3d(rget(x, ti));
                    const float3 ab = b - a;
                    const float l = len(ab);
                    of = a;
                    d = ab * (1.0f / l);
                    tmax = l - P.ray_eps;
                } else {
                    if (tmode == TR_REPROJ) {
                        const double3 v = (rget(x, ti) + tod(rget(dq, ti)) * (double)beta) - to;
                        const double l2 = ddot(v, v);
                        if (!(l2 > 0.0)) { tcode = 3 | (ti << 4); has = false; }
                        else tdd = v * rsqrt(l2);
                        hint = rget(prim, ti);
                    } else if (ti > 0) {
                        if (!scatter_dir<GL>(S, tdd, tpp, tps, to, (tres >> (ti - 1)) & 1u, g.seed, P.walk_id_base + w,
                                         ti - 1)) {
                            tcode = 4 | (ti << 4);
                            has = false;
                        }
                    }
                    of = f3d(to);
                    d = nrmz(f3d(tdd));
                }
                if (!has) ti = -1;
            }
            // 2. slot = rank among the block's rays
            const unsigned bal = __ballot_sync(MPG_FULL, has);
            if (lane == 0) s_wcnt[warp] = __popc(bal);
            __syncthreads();
            int rbase = 0, M = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int c = s_wcnt[q];
                rbase += q < warp ? c : 0;
                M += c;
            }
            const int slot = rbase + __popc(bal & ((1u << lane) - 1u));
            if (has) {
                s_ro[slot] = make_float4(of.x, of.y, of.z, tmax);
                s_rd[slot] = make_float4(d.x, d.y, d.z, __int_as_float(tmode == TR_VIS ? 1 : 0));
                s_rh[slot] = hint;
            }
            __syncthreads();
            // 3. the first M threads trace the M rays
            if ((int)threadIdx.x < M) {
                const float4 ro = s_ro[threadIdx.x], rd = s_rd[threadIdx.x];
                const bool vis = __float_as_int(rd.w) != 0;
                Hit h;
                ls.rays++;
                const bool hit = trace<W>(S, xyz(ro), xyz(rd), P.ray_eps, ro.w, !vis, vis, h, ls,
                                          vis ? -1 : s_rh[threadIdx.x], top);
                s_hp[threadIdx.x] = make_float4(h.p.x, h.p.y, h.p.z, 0.f);
                s_hs[threadIdx.x] = make_int2(hit ? h.prim : -3, h.surf);
            }
            __syncthreads();
            // 4. consume the hit (bottom of the trace_chain loop body)
            if (has) {
                const int2 hs = s_hs[slot];
                const bool hit = hs.x != -3;
                if (tmode == TR_VIS) {
                    if (hit) { tcode = 5; ti = -1; }
                    else if (++ti >= tnr) ti = -1;
                } else if (!hit) {
                    tcode = 1 | (ti << 4);
                    ti = -1;
                } else if (tmode == TR_REPROJ && hs.y != (int)((sreq >> (4 * ti)) & 15u)) {
                    tcode = 2 | (ti << 4);
                    ti = -1;
                } else {
                    if (tmode == TR_DEDUCE) {
                        uint32_t bit = (bits >> ti) & 1u;
                        const int mat = S.surf[hs.y].mat;
                        if (!learned && mat == 0) bit = 0u;
                        if (bit && mat != 1) { tcode = 4 | (ti << 4); ti = -1; }
                        else tres |= bit << ti;
                    }
                    if (ti >= 0) {
                        const float4 hp = s_hp[slot];
                        int hprim = hs.x;
                        const double3 yi = refine_hit(S, hprim, hs.y, to,
                                                      tmode == TR_DEDUCE ? to + tdd
                                                                         : rget(x, ti) + tod(rget(dq, ti)) * (double)beta,
                                                      f3(hp.x, hp.y, hp.z));
                        rset(y, ti, yi);
                        rset(yp, ti, hprim);
                        rset(ys, ti, hs.y);
                        tpp = hprim;
                        tps = hs.y;
                        to = yi;
                        if (++ti >= tnr) ti = -1;
                    }
                }
            }
        }
        if (tracing) {
            const bool ded = tmode == TR_DEDUCE;
            const int mode = tmode;
            const int why = tcode;
            bool ok = why == 0;
            MPG_TRACE_TAIL
        }
        }

        // ---- Newton system / step ------------------------------------------
        if (phase == PH_SOLVE) {
            if (fresh) {
                fresh = false;
                c_vtx += k;
                float cm = 0.f;
                bool singular = false;
                R Di[KMAX][4], Ub[KMAX][4];      // transient: D'^-1_i, U_i of the block-Thomas sweep
                V3<R> sg[KMAX], tg[KMAX];          // transient: tangent frames of the step
                int r = newton_system<KMAX, R, GL>(S, g.seed, P.walk_id_base + w, k, tau, xD, xL, x, prim, surf, P.tol, Di, Ub,
                                               sg, tg, dq, singular, cm);
                if (P.dbg && trial == 0 && w < P.n_dbg && 2 * it + 1 < P.dbg_stride) {
                    P.dbg[w * P.dbg_stride + 2 * it] = cm;
                    P.dbg[w * P.dbg_stride + 2 * it + 1] = beta;
                }
                if (r == 1) {
                    end_status = ST_CONVERGED;
                    phase = PH_END;
                    if (trial == 0) {
                        // a converged primary: sides (R8; BAD_SIDE precedes OCCLUDED), kappa and the
                        // analytic GGT from this sweep's blocks (R11, R12), then its k+1 visibility
                        // segments in the next trace phase (PH_VIS)
                        const DLight &L = S.light[lid];
                        float kap;
                        R DL[4];
                        if (!post_sweep<KMAX, R, GL>(S, g.seed, P.walk_id_base + w, L, k, tau, xD, xL, x, prim, surf, true, kap,
                                                 DL)) {
                            end_status = ST_BAD_SIDE;
                        } else {
                            const float3 nD = xyz(__ldg(P.nD + (uint32_t)w / (uint32_t)P.spp));
                            Gc = singular ? 0.0f : ggt_from_blocks<KMAX, R>(k, xD, nD, x, Di, Ub, sg, tg, DL);
                            float Le = L.emit;
                            if (L.kind == 1 && !(dot(f3d(x[k - 1]) - xL, L.n) > 0.0f)) Le = 0.0f;
                            Tc = kap * Gc * Le;
                            phase = PH_VIS;
                        }
                    }
                }
                else if (r == 2) { end_status = ST_DEGENERATE; phase = PH_END; }
            }
            if (phase == PH_SOLVE) {
                if (it >= ((k >= 3 && P.max_iters_long > 0) ? P.max_iters_long : P.max_iters)) {
                    end_status = ST_MAXITER;
                    phase = PH_END;
                }
                else phase = PH_REPROJ;
            }
        }

        // ---- end of an attempt ---------------------------------------------
        if constexpr (MPG_SVC_ALL || CMP || KMAX <= 2) {   // (fixed long chains have few boundaries per pass: measured no gain)
            // serve now? (always in the tail: idle lanes are waiting for exactly this work)
            const int nwait = __popc(__ballot_sync(MPG_FULL, phase == PH_END || phase == PH_FETCH || phase == PH_SEED));
            svc = nwait >= (int)P.svc_min || ++svc_since >= (int)P.svc_wait || drained || nwait == 0;
            if (svc) svc_since = 0;
        }
        if (phase == PH_END && svc) {
            c_newton += it;
            int st = end_status;
            if (trial == 0) {
                float G = 0.f, T = 0.f;
                if (st == ST_CONVERGED) {
                    // visibility: k+1 any-hit segments against all surfaces, V = 0 -> G = T = 0
                    if (occluded) st = ST_OCCLUDED;
                    else { G = Gc; T = Tc; }
                }
                if (st != ST_SEED_FAIL && st != ST_INACTIVE) {
#pragma unroll
                    for (int i = 0; i < KMAX; i++) {
                        if (i >= k) break;
                        int pid = prim[i] >= 0 ? __float_as_int(__ldg(S.tpos + TSTRIDE * prim[i]).w) : -1;
                        MPG_CHECK(w >= 0 && w < P.n && i < KMAX);
                        P.chain[(int64_t)i * P.n + w] = make_float4((float)x[i].x, (float)x[i].y, (float)x[i].z, __int_as_float(pid));
                    }
                }
                P.status[w] = (uint8_t)st;
                P.iters[w] = (uint16_t)it;
                P.G[w] = G;
                P.T[w] = T;
                if (P.out_ctype) P.out_ctype[w] = (uint16_t)((uint32_t)k | (tau << 4));
                atomicAdd(&s_stats[SS_STATUS0 + st], 1u);
                atomicAdd(&s_stats[SS_PRIM_IT], (unsigned)it);
                atomicAdd(&s_stats[SS_WALKS], 1u);
                if (st == ST_CONVERGED || st == ST_OCCLUDED) atomicAdd(&s_stats[SS_CONV], 1u);
                if (st == ST_CONVERGED && T > 0.0f && P.trials_on) {
                    Tprim = T;
                    pk = k;
                    ptau = tau;
                    psurf = 0;
#pragma unroll
                    for (int i = 0; i < KMAX; i++) {
                        if (i >= k) break;
                        psurf |= (uint32_t)(surf[i] & 15) << (4 * i);
                    }
                    if (P.psurf_out) P.psurf_out[w] = psurf;
                    if (queue_drained(P, drained) && P.items && hard_publish(P, w, psurf, pk, ptau, 0u, seq_only))
                        phase = PH_FETCH;
                    else {
                        trial = 1;
                        phase = PH_SEED;
                    }
                } else {
                    P.trials[w] = 0;
                    P.w[w] = 0.0f;
                    walk_resolved(P);
                    phase = PH_FETCH;
                }
            } else {
                bool same = false;
                float kdummy;
                R DLdummy[4];
                if (st == ST_CONVERGED && k == pk && tau == ptau &&
                    post_sweep<KMAX, R, GL>(S, g.seed, P.walk_id_base + w, S.light[lid], k, tau, xD, xL, x, prim, surf, false,
                                        kdummy, DLdummy)) {
                    same = true;
#pragma unroll
                    for (int i = 0; i < KMAX; i++) {
                        if (i >= k) break;
                        float4 c = __ldcg(P.chain + (int64_t)i * P.n + w);
                        float3 dd = f3d(x[i]) - xyz(c);
                        if ((int)((psurf >> (4 * i)) & 15u) != (surf[i] & 15) || !(len(dd) < P.same_eps)) same = false;
                    }
                }
                if (item_e >= 0) {
                    // one item of a batch: the last one to finish decides the entry
                    const uint32_t e = (uint32_t)item_e;
                    if (same) atomicMin(P.e_best + e, trial);
                    __threadfence();
                    unsigned left = atomicSub(P.e_pending + e, 1u) - 1u;
                    phase = PH_FETCH;
                    if (left == 0) {
                        __threadfence();
                        const uint32_t b = *(volatile uint32_t *)(P.e_best + e);
                        const uint32_t issued = __ldcg(P.e_issued + e);
                        if (b != HARD_NONE) {
                            trial_finalize(P, w, b, false, s_stats);
                            walk_resolved(P);
                        } else if (issued >= P.k_max) {
                            trial_finalize(P, w, P.k_max, true, s_stats);
                            walk_resolved(P);
                        } else {
                            const unsigned backlog = *(volatile unsigned *)&P.th->item_tail -
                                                     *(volatile unsigned *)&P.th->item_head;
                            const uint32_t g = (int)backlog < (int)P.idle_backlog && queue_drained(P, drained) ? P.item_grow_idle
                                                                                             : P.item_grow;
                            const uint32_t B = min(__ldcg(P.e_batch + e) << g, P.k_max - issued);
                            P.e_batch[e] = B;
                            P.e_pending[e] = B;
                            P.e_issued[e] = issued + B;
                            __threadfence();
                            if (!items_push(P, e, issued + 1, B)) {
                                // ring full: continue this walk's trials sequentially here
                                P.e_pending[e] = 0;
                                item_e = -1;
                                seq_only = true;
                                trial = issued + 1;
                                phase = PH_SEED;
                            }
                        }
                    }
                } else if (same || trial >= P.k_max) {
                    trial_finalize(P, w, trial, !same, s_stats);
                    walk_resolved(P);
                    phase = PH_FETCH;
                } else {
                    // hand the remaining trials to parallel items after local_trials
                    // sequential ones, or at once when the primary queue is exhausted
                    // (idle lanes are then waiting for exactly this work)
                    if ((trial >= P.local_trials || queue_drained(P, drained)) && !seq_only && P.items &&
                        hard_publish(P, w, psurf, pk, ptau, trial, seq_only))
                        phase = PH_FETCH;
                    else {
                        trial++;
                        phase = PH_SEED;
                    }
                }
            }
        }
    }

    // ---- stats reduction ----------------------------------------------------
    unsigned long long v[6] = {c_newton, c_attempts, (unsigned long long)ls.rays + s_rays[threadIdx.x], ls.nodes,
                               ls.tris, c_vtx};
#pragma unroll
    for (int j = 0; j < 6; j++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(MPG_FULL, v[j], o);
    }
    if (lane == 0) {
        // work counters per warp straight into the 64-bit global stats
        if (P.stats) {
            atomicAdd(P.stats + SS_NEWTON, v[0]);
            atomicAdd(P.stats + SS_ATTEMPTS, v[1]);
            atomicAdd(P.stats + SS_RAYS, v[2]);
            atomicAdd(P.stats + SS_NODES, v[3]);
            atomicAdd(P.stats + SS_TRIS, v[4]);
            atomicAdd(P.stats + SS_VTX, v[5]);
        }
    }
    __syncthreads();
    if (P.stats)
        for (int i = threadIdx.x; i < SS_N; i += blockDim.x)
            if (s_stats[i]) atomicAdd(P.stats + i, (unsigned long long)s_stats[i]);
}
#undef MPG_TRACE_TAIL
