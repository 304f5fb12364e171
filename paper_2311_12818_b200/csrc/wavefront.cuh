// wavefront.cuh -- wavefront formulation of the batched manifold walk (default path).
//
// The megakernel (walk.cuh) keeps one chain per lane, so a warp waits for the
// slowest of 32 chained ray traversals each Newton iteration: ncu measured 4.6
// active threads per warp.  Here the walk state lives in S "slots" in global
// memory (SoA) and every Newton iteration is one *wave* of four kernels, run
// by a CUDA-graph while loop (device-side cudaGraphSetConditional, no host sync):
//
//   k_wf_trace   persistent, per-lane job fetch (Aila & Laine 2009): a job is
//                the k sequential rays of one slot (deduction, Eq. 6, or
//                ray-traced reprojection); a lane that finishes its job takes
//                the next one, so traversal runs with full warps regardless of
//                per-ray trip counts.  While-while traversal, postponed leaves.
//   k_wf_update  one thread per traced slot: accept/halve (R6), Newton system
//                fused with block-Thomas (R1-R4, R7), step; at the end of an
//                attempt: sides (R8), visibility, kappa, G, T (Eq. 2); trials
//                (Eq. 15): sequential up to LOCAL_TRIALS, then the walk becomes
//                a "hard entry" whose further trials run as independent items
//                in doubling batches; k = min successful trial (exactly the
//                sequential geometric count).  Freed slots go to a free stack.
//   k_wf_plan    one thread: snapshot of free slots / pending items / queue,
//                assignment plan, loop condition.
//   k_wf_refill  assigns hard-entry trial items, then new primary walks, to
//                free slots (deterministic from the plan, no contention).
#pragma once
#include "walk.cuh"

#define WF_LOCAL_TRIALS 4u
#define WF_BATCH0 4u
#define WF_NONE 0xffffffffu
// slot flag bits (s_flags)
#define F_DEDUCE (1u << 16)
#define F_FAIL (1u << 17)
#define F_ITEM (1u << 18)
#define F_SEEDFAIL (1u << 19)
#define F_SEQ (1u << 20)      // hard entry continued sequentially in this slot (item list full)
#define F_IT_MASK 0xffffu

struct WFHeader {                 // device counters (in the workspace)
    unsigned long long queue;     // next primary walk
    unsigned int wave;            // parity of the current ray list
    unsigned int list_count[2];
    unsigned int free_top;        // free-slot stack size
    unsigned int n_entries;       // hard entries published
    unsigned int item_head, item_tail;
    // plan (written by k_wf_plan, read by k_wf_refill)
    unsigned int plan_free, plan_items, plan_prims, plan_list;
    unsigned long long plan_queue0;
    unsigned int plan_item0;
    unsigned int trace_cursor;    // job cursor of k_wf_trace (reset by k_wf_plan)
    unsigned int more;            // work remains after this wave (host-loop mode)
};

struct WFParams {
    // inputs / outputs (as the megakernel)
    const float4 *xD, *nD;
    int64_t n;
    int spp;
    const float4 *seed_xL, *seed_tgt;
    const int *seed_bin;
    float4 *chain;
    uint8_t *status;
    uint16_t *iters;
    float *G, *T, *w;
    uint32_t *trials;
    unsigned long long *stats;
    int max_iters, trials_on;
    uint32_t k_max;
    float tol, beta0, same_eps, ray_eps;
    uint64_t walk_id_base;
    // wavefront state
    WFHeader *hdr;
    uint32_t S;                   // slots
    uint32_t *list[2];
    uint32_t *free_stack;
    int32_t *s_walk;
    uint32_t *s_trial, *s_flags, *s_surf, *s_ysurf, *s_psurf;
    int32_t *s_entry;
    float *s_beta;
    float4 *s_tgt;
    double4 *s_x, *s_y;           // [k][S] chain / traced vertices (fp64 positions, w = prim)
    float4 *s_dq;                 // [k][S] Newton step directions
    uint32_t H;                   // hard entry capacity
    int32_t *e_walk;
    uint32_t *e_psurf, *e_best, *e_issued, *e_pending, *e_batch;
    uint32_t C;                   // item capacity
    int32_t *it_entry;
    uint32_t *it_trial;
    cudaGraphConditionalHandle cond;
    int use_cond;                 // 1: inside the CUDA-graph while loop; 0: host-driven waves (profiling)
};

// --------------------------------------------------------------------------
// shared helpers
// --------------------------------------------------------------------------
__device__ __forceinline__ void wf_append(const WFParams &P, uint32_t lst, uint32_t slot) {
    // warp-aggregated append to ray list `lst`
    unsigned m = __activemask();
    int leader = __ffs(m) - 1;
    int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(&P.hdr->list_count[lst], (unsigned)__popc(m));
    base = __shfl_sync(m, base, leader);
    P.list[lst][base + __popc(m & ((1u << lane) - 1u))] = slot;
}

__device__ __forceinline__ void wf_free(const WFParams &P, uint32_t slot) {
    unsigned m = __activemask();
    int leader = __ffs(m) - 1;
    int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(&P.hdr->free_top, (unsigned)__popc(m));
    base = __shfl_sync(m, base, leader);
    P.free_stack[base + __popc(m & ((1u << lane) - 1u))] = slot;
    P.s_walk[slot] = -1;
}

// start an attempt (seed) in `slot`: deduction target for (walk, trial)
__device__ __forceinline__ void wf_seed(const DScene &S, const SeedCtx &g, const WFParams &P, uint32_t slot,
                                        int64_t w, uint32_t trial, uint32_t extra_flags) {
    float3 tgt = f3(0.f, 0.f, 0.f);
    bool ok;
    if (trial == 0) {
        ok = __ldg(P.seed_bin + w) != -2;
        tgt = xyz(__ldg(P.seed_tgt + w));
    } else {
        SeedRes sr;
        ok = seed_target(S, g, P.walk_id_base + w, trial, xyz(__ldg(P.xD + w / P.spp)), sr);
        tgt = sr.tgt;
    }
    P.s_walk[slot] = (int32_t)w;
    P.s_trial[slot] = trial;
    P.s_flags[slot] = F_DEDUCE | extra_flags | (ok ? 0u : F_SEEDFAIL);
    P.s_tgt[slot] = make_float4(tgt.x, tgt.y, tgt.z, 0.f);
}

// --------------------------------------------------------------------------
// init: slots 0..min(S,n)-1 <- walks 0..; list[0] = those slots
// --------------------------------------------------------------------------
template <int KMAX>
__global__ void k_wf_init(const DScene S, const SeedCtx g, const WFParams P) {
    uint32_t s0 = (uint32_t)min((int64_t)P.S, P.n);
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < P.S; s += gridDim.x * blockDim.x) {
        if (s < s0) {
            wf_seed(S, g, P, s, (int64_t)s, 0u, 0u);
            P.list[0][s] = s;
        } else {
            P.s_walk[s] = -1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        WFHeader *h = P.hdr;
        h->queue = s0;
        h->wave = 0;
        h->list_count[0] = s0;
        h->list_count[1] = 0;
        h->free_top = 0;
        h->n_entries = 0;
        h->item_head = h->item_tail = 0;
        h->trace_cursor = 0;
    }
}

// --------------------------------------------------------------------------
// trace: persistent, per-lane job fetch, while-while traversal
// --------------------------------------------------------------------------
template <int KMAX>
__global__ void __launch_bounds__(128) k_wf_trace(const DScene S, const SeedCtx g, const WFParams P) {
    __shared__ unsigned long long s_acc[3];
    if (threadIdx.x < 3) s_acc[threadIdx.x] = 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned par = *(volatile unsigned int *)&P.hdr->wave & 1u;
    const uint32_t *list = P.list[par];
    const unsigned count = *(volatile unsigned int *)&P.hdr->list_count[par];
    const int k = g.k;
    const uint32_t tau = g.tau;
    const float eps = P.ray_eps;
    const int SENT = 0x7fffffff, NONE = 0;
    // job / ray state
    int slot = -1, i = 0;
    bool deduce = false, active = false, job_done = false;
    uint32_t surf_req = 0, ysurf = 0;
    float3 xD = f3(0, 0, 0), o = f3(0, 0, 0), d = f3(0, 0, 0);
    double3 od = make_double3(0, 0, 0), dd = make_double3(0, 0, 0), q = make_double3(0, 0, 0);
    int pprim = -1, psurf_ = -1; // previous hit (for deduction scattering)
    float beta = 1.f;
    RayW r;
    r.o = o; r.d = d; r.idir = d; r.kx = 0; r.ky = 1; r.kz = 2; r.Sx = r.Sy = r.Sz = 0.f;
    float best = 0.f, bb0 = 0.f, bb1 = 0.f, bb2 = 0.f;
    int bprim = -2, bsurf = -1;
    float3 bp = f3(0, 0, 0);
    int node = SENT, leaf = NONE, sp = 0;
    int stack[64];
    LaneStats ls = {0u, 0u, 0u};
    unsigned int *cursor = &P.hdr->trace_cursor;  // jobs = entries of the current ray list

    while (true) {
        // ---- lanes without a job fetch one (warp-aggregated) ----
        unsigned need = __ballot_sync(MPG_FULL, slot < 0 && !job_done);
        if (need) {
            int leader = __ffs(need) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(cursor, (unsigned)__popc(need));
            base = __shfl_sync(MPG_FULL, base, leader);
            if (slot < 0 && !job_done) {
                unsigned idx = base + __popc(need & ((1u << lane) - 1u));
                if (idx < count) {
                    slot = (int)list[idx];
                    uint32_t fl = P.s_flags[slot];
                    deduce = (fl & F_DEDUCE) != 0;
                    int64_t w = P.s_walk[slot];
                    xD = xyz(__ldg(P.xD + w / P.spp));
                    i = 0;
                    ysurf = 0;
                    if (fl & F_SEEDFAIL) {
                        P.s_flags[slot] = fl | F_FAIL;
                        slot = -1;
                    } else {
                        surf_req = P.s_surf[slot];
                        beta = P.s_beta[slot];
                        if (deduce) {
                            double3 v = d3f(xyz(P.s_tgt[slot])) - d3f(xD);
                            double l2 = ddot(v, v);
                            dd = l2 > 0.0 ? v * rsqrt(l2) : make_double3(0, 0, 0);
                        }
                        active = false; // ray 0 set up below
                    }
                } else {
                    job_done = true; // queue drained
                }
            }
        }
        if (__all_sync(MPG_FULL, slot < 0 && job_done)) break;

        // ---- set up ray i of the job (if not yet active) ----
        if (slot >= 0 && !active) {
            bool ok = true;
            if (i == 0) od = d3f(xD);
            if (deduce) {
                if (i > 0) ok = scatter_dir(S, dd, pprim, psurf_, f3d(od), (tau >> (i - 1)) & 1u);
                else ok = ddot(dd, dd) > 0.0;
            } else {
                double4 x4 = P.s_x[(size_t)i * P.S + slot];
                float4 dq4 = P.s_dq[(size_t)i * P.S + slot];
                q = make_double3(x4.x + (double)dq4.x * beta, x4.y + (double)dq4.y * beta, x4.z + (double)dq4.z * beta);
                double3 v = q - od;
                double l2 = ddot(v, v);
                ok = l2 > 0.0;
                if (ok) dd = v * rsqrt(l2);
            }
            o = f3d(od);
            d = nrmz(f3d(dd));
            if (!ok) {
                P.s_flags[slot] |= F_FAIL;
                slot = -1;
            } else {
                ls.rays++;
                best = 3.0e38f; bprim = -2; bsurf = -1;
                for (int s = 0; s < S.n_surf; s++) {
                    const DSurf &f = S.surf[s];
                    if (f.kind == 2 || f.mat == 2) continue;
                    float t; float3 p; bool hit;
                    if (f.kind == 0) hit = sphere_hit(o, d, f.center, f.radius, eps, best, t, p);
                    else { hit = quad_hit(o, d, f.origin, f.eu, f.ev, eps, best, t); p = o + d * t; }
                    if (hit) { best = t; bprim = -1; bsurf = s; bp = p; }
                }
                if (S.n_tri > 0) {
                    ray_setup(r, o, d);
                    node = 0; leaf = NONE; stack[0] = SENT; sp = 1;
                } else {
                    node = SENT; leaf = NONE;
                }
                active = true;
            }
        }

        // ---- traversal: while-while with postponed leaves ----
        if (slot >= 0 && active) {
            while (node >= 0 && node != SENT) {
                ls.nodes++;
                const float4 *nd = S.nodes + 4 * node;
                float4 a = __ldg(nd), b = __ldg(nd + 1), c = __ldg(nd + 2);
                int4 ch = __ldg(reinterpret_cast<const int4 *>(nd + 3));
                float tx0 = (a.x - o.x) * r.idir.x, tx1 = (a.w - o.x) * r.idir.x;
                float ty0 = (a.y - o.y) * r.idir.y, ty1 = (b.x - o.y) * r.idir.y;
                float tz0 = (a.z - o.z) * r.idir.z, tz1 = (b.y - o.z) * r.idir.z;
                float n0 = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), eps));
                float f0 = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), best));
                float sx0 = (b.z - o.x) * r.idir.x, sx1 = (c.y - o.x) * r.idir.x;
                float sy0 = (b.w - o.y) * r.idir.y, sy1 = (c.z - o.y) * r.idir.y;
                float sz0 = (c.x - o.z) * r.idir.z, sz1 = (c.w - o.z) * r.idir.z;
                float n1 = fmaxf(fmaxf(fminf(sx0, sx1), fminf(sy0, sy1)), fmaxf(fminf(sz0, sz1), eps));
                float f1 = fminf(fminf(fmaxf(sx0, sx1), fmaxf(sy0, sy1)), fminf(fmaxf(sz0, sz1), best));
                bool h0 = n0 <= f0, h1 = n1 <= f1;
                if (h0 && h1) {
                    bool swp = n1 < n0;
                    node = swp ? ch.y : ch.x;
                    stack[sp++] = swp ? ch.x : ch.y;
                } else if (h0) node = ch.x;
                else if (h1) node = ch.y;
                else node = stack[--sp];
                if (node < 0 && leaf == NONE) { leaf = node; node = stack[--sp]; }
                if (!__any_sync(__activemask(), leaf == NONE)) break;
            }
            while (leaf != NONE) {
                int v = ~leaf;
                int start = v >> 3, cnt = (v & 7) + 1;
                for (int j = start; j < start + cnt; j++) {
                    ls.tris++;
                    float4 p0 = __ldg(S.tpos + 3 * j), p1 = __ldg(S.tpos + 3 * j + 1), p2 = __ldg(S.tpos + 3 * j + 2);
                    if (__float_as_int(p2.w) == 0) continue;
                    float t, c0, c1, c2;
                    if (tri_hit(r, xyz(p0), xyz(p1), xyz(p2), eps, best, t, c0, c1, c2)) {
                        best = t; bprim = j; bsurf = __float_as_int(p1.w);
                        bb0 = c0; bb1 = c1; bb2 = c2;
                    }
                }
                leaf = NONE;
                if (node < 0) { leaf = node; node = stack[--sp]; }
            }
            // ---- ray finished? ----
            if (node == SENT && leaf == NONE) {
                active = false;
                bool ok = bsurf >= 0 && (deduce || bsurf == (int)((surf_req >> (4 * i)) & 15u));
                if (!ok) {
                    P.s_flags[slot] |= F_FAIL;
                    slot = -1;
                } else {
                    float3 pf;
                    if (bprim >= 0) {
                        float3 v0 = xyz(__ldg(S.tpos + 3 * bprim)), v1 = xyz(__ldg(S.tpos + 3 * bprim + 1)),
                               v2 = xyz(__ldg(S.tpos + 3 * bprim + 2));
                        pf = v0 * bb0 + v1 * bb1 + v2 * bb2;
                    } else pf = bp;
                    double3 y = refine_hit(S, bprim, bsurf, od, deduce ? od + dd : q, pf);
                    P.s_y[(size_t)i * P.S + slot] = make_double4(y.x, y.y, y.z, (double)bprim);
                    ysurf |= (uint32_t)(bsurf & 15) << (4 * i);
                    pprim = bprim; psurf_ = bsurf;
                    od = y;
                    i++;
                    if (i >= k) {
                        P.s_ysurf[slot] = ysurf;
                        P.s_flags[slot] &= ~F_FAIL;
                        slot = -1;
                    }
                }
            }
        }
    }
    // stats
    unsigned long long v3[3] = {ls.rays, ls.nodes, ls.tris};
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v3[j] += __shfl_down_sync(MPG_FULL, v3[j], off);
    if (lane == 0) {
        atomicAdd(&s_acc[0], v3[0]);
        atomicAdd(&s_acc[1], v3[1]);
        atomicAdd(&s_acc[2], v3[2]);
    }
    __syncthreads();
    if (threadIdx.x == 0 && P.stats) {
        atomicAdd(P.stats + SS_RAYS, s_acc[0]);
        atomicAdd(P.stats + SS_NODES, s_acc[1]);
        atomicAdd(P.stats + SS_TRIS, s_acc[2]);
    }
}

// --------------------------------------------------------------------------
// hard entries: finalize / next batch
// --------------------------------------------------------------------------
__device__ __forceinline__ void wf_finalize_walk(const WFParams &P, int64_t w, uint32_t kk, bool truncated,
                                                 unsigned long long *s_stats) {
    P.trials[w] = kk;
    P.w[w] = P.T[w] * (float)kk / __ldg(P.seed_xL + w).w;
    atomicAdd(&s_stats[SS_TRIALS], (unsigned long long)kk);
    if (truncated) atomicAdd(&s_stats[SS_TRUNC], 1ull);
}

// append `cnt` items (e, t0..t0+cnt-1); returns false if the item list is full
__device__ __forceinline__ bool wf_push_items(const WFParams &P, uint32_t e, uint32_t t0, uint32_t cnt) {
    unsigned base = atomicAdd(&P.hdr->item_tail, cnt);
    if (base + cnt > P.C) return false;
    for (uint32_t j = 0; j < cnt; j++) {
        P.it_entry[base + j] = (int32_t)e;
        P.it_trial[base + j] = t0 + j;
    }
    return true;
}

// --------------------------------------------------------------------------
// update: one thread per traced slot
// --------------------------------------------------------------------------
template <int KMAX>
__global__ void __launch_bounds__(128) k_wf_update(const DScene S, const SeedCtx g, const WFParams P) {
    __shared__ unsigned long long s_stats[SS_N];
    for (int j = threadIdx.x; j < SS_N; j += blockDim.x) s_stats[j] = 0ull;
    __syncthreads();
    const unsigned par = *(volatile unsigned int *)&P.hdr->wave & 1u;
    const uint32_t *list = P.list[par];
    const unsigned count = *(volatile unsigned int *)&P.hdr->list_count[par];
    const unsigned nxt = par ^ 1u;
    const int k = g.k;
    const uint32_t tau = g.tau;
    uint32_t c_newton = 0, c_vtx = 0, c_att = 0, c_rays = 0;
    LaneStats ls = {0u, 0u, 0u};

    for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < count; idx += gridDim.x * blockDim.x) {
        const uint32_t slot = list[idx];
        uint32_t fl = P.s_flags[slot];
        const int64_t w = P.s_walk[slot];
        uint32_t trial = P.s_trial[slot];
        int it = (int)(fl & F_IT_MASK);
        float beta = P.s_beta[slot];
        bool deduce = fl & F_DEDUCE, failed = fl & F_FAIL;
        double3 x[KMAX];
        V3<float> sg[KMAX], tg[KMAX], dq[KMAX];
        int prim[KMAX], surf[KMAX];
        float Di[KMAX][4], Ub[KMAX][4];
        uint32_t sp_ = failed ? P.s_surf[slot] : P.s_ysurf[slot];
        const double4 *src = failed ? P.s_x : P.s_y;
#pragma unroll
        for (int j = 0; j < KMAX; j++) {
            if (j >= k) { x[j] = make_double3(0, 0, 0); sg[j] = tg[j] = dq[j] = mk3<float>(0, 0, 0); prim[j] = -1; surf[j] = 0; continue; }
            double4 v = src[(size_t)j * P.S + slot];
            x[j] = make_double3(v.x, v.y, v.z);
            prim[j] = (int)v.w;
            surf[j] = (int)((sp_ >> (4 * j)) & 15u);
            sg[j] = tg[j] = dq[j] = mk3<float>(0, 0, 0);
        }
        int end = -1; // attempt end status
        bool fresh = false;
        if (deduce) {
            if (failed) end = ST_SEED_FAIL;
            else { it = 0; beta = P.beta0; fresh = true; }
        } else if (failed) {
            beta *= 0.5f; it++;
        } else {
            beta = fminf(1.0f, 2.0f * beta); it++; fresh = true;
        }
        const float3 xD = xyz(__ldg(P.xD + w / P.spp));
        const float4 l4 = __ldg(P.seed_xL + w);
        const float3 xL = xyz(l4);
        bool singular = false;
        if (end < 0) {
            if (fresh) {
                c_vtx += k;
                float cm;
                int rr = newton_system<KMAX, float>(S, k, tau, xD, xL, x, prim, surf, P.tol, Di, Ub, sg, tg, dq, singular, cm);
                if (rr == 1) end = ST_CONVERGED;
                else if (rr == 2) end = ST_DEGENERATE;
                else {
#pragma unroll
                    for (int j = 0; j < KMAX; j++)
                        if (j < k) P.s_dq[(size_t)j * P.S + slot] = make_float4(dq[j].x, dq[j].y, dq[j].z, 0.f);
                }
            }
            if (end < 0 && it >= P.max_iters) end = ST_MAXITER;
        }
        if (end < 0) {
            // continue: reprojection next wave
            if (fresh) {
#pragma unroll
                for (int j = 0; j < KMAX; j++)
                    if (j < k) P.s_x[(size_t)j * P.S + slot] = make_double4(x[j].x, x[j].y, x[j].z, (double)prim[j]);
                P.s_surf[slot] = sp_;
            }
            P.s_beta[slot] = beta;
            P.s_flags[slot] = (fl & (F_ITEM | F_SEQ)) | (uint32_t)it;
            wf_append(P, nxt, slot);
            continue;
        }
        // ---------------- attempt ended ----------------
        c_newton += it;
        c_att++;
        int lid = 0;
        if (S.n_light > 1) lid = (int)uidx(rng_draw(g.seed, P.walk_id_base + w, 0u, 0u).z, (uint32_t)S.n_light);
        if (trial == 0) {
            float Gv = 0.f, Tv = 0.f;
            int st = end;
            if (st == ST_CONVERGED) {
                const DLight &L = S.light[lid];
                float kap, DL[4];
                if (!post_sweep<KMAX, float>(S, L, k, tau, xD, xL, x, prim, surf, true, kap, DL)) st = ST_BAD_SIDE;
                else {
                    bool vis = true;
                    float3 a = xD;
#pragma unroll 1
                    for (int j = 0; j <= k; j++) {
                        float3 b = xL;
#pragma unroll
                        for (int jj = 0; jj < KMAX; jj++)
                            if (jj == j) b = f3d(x[jj]);
                        float3 dd = b - a;
                        float l = len(dd);
                        Hit hh;
                        if (trace<true>(S, a, dd * (1.0f / l), P.ray_eps, l - P.ray_eps, false, hh, ls)) { vis = false; break; }
                        a = b;
                    }
                    if (!vis) st = ST_OCCLUDED;
                    else {
                        Gv = singular ? 0.0f : ggt_from_blocks<KMAX, float>(k, xD, xyz(__ldg(P.nD + w / P.spp)), x, Di, Ub, sg, tg, DL);
                        float Le = L.emit;
                        if (L.kind == 1 && !(dot(f3d(x[k - 1]) - xL, L.n) > 0.0f)) Le = 0.0f;
                        Tv = kap * Gv * Le;
                    }
                }
            }
            if (st != ST_SEED_FAIL) {
#pragma unroll
                for (int j = 0; j < KMAX; j++) {
                    if (j >= k) break;
                    int pid = prim[j] >= 0 ? __float_as_int(__ldg(S.tpos + 3 * prim[j]).w) : -1;
                    P.chain[(int64_t)j * P.n + w] = make_float4((float)x[j].x, (float)x[j].y, (float)x[j].z, __int_as_float(pid));
                }
            }
            P.status[w] = (uint8_t)st;
            P.iters[w] = (uint16_t)it;
            P.G[w] = Gv;
            P.T[w] = Tv;
            atomicAdd(&s_stats[SS_STATUS0 + st], 1ull);
            atomicAdd(&s_stats[SS_PRIM_IT], (unsigned long long)it);
            atomicAdd(&s_stats[SS_WALKS], 1ull);
            if (st == ST_CONVERGED || st == ST_OCCLUDED) atomicAdd(&s_stats[SS_CONV], 1ull);
            if (st == ST_CONVERGED && Tv > 0.0f && P.trials_on) {
                P.s_psurf[slot] = sp_;
                wf_seed(S, g, P, slot, w, 1u, 0u);
                wf_append(P, nxt, slot);
            } else {
                P.trials[w] = 0;
                P.w[w] = 0.0f;
                wf_free(P, slot);
            }
            continue;
        }
        // trial attempt: same chain as the primary?
        const bool item = fl & F_ITEM;
        const uint32_t e = item ? (uint32_t)P.s_entry[slot] : 0u;
        const uint32_t psurf = item ? P.e_psurf[e] : P.s_psurf[slot];
        bool same = false;
        if (end == ST_CONVERGED) {
            float kd, DLd[4];
            if (post_sweep<KMAX, float>(S, S.light[lid], k, tau, xD, xL, x, prim, surf, false, kd, DLd)) {
                same = true;
#pragma unroll
                for (int j = 0; j < KMAX; j++) {
                    if (j >= k) break;
                    float3 dd = f3d(x[j]) - xyz(P.chain[(int64_t)j * P.n + w]);
                    if ((int)((psurf >> (4 * j)) & 15u) != surf[j] || !(len(dd) < P.same_eps)) same = false;
                }
            }
        }
        if (item && !(fl & F_SEQ)) {
            if (same) atomicMin(P.e_best + e, trial);
            __threadfence();
            unsigned left = atomicSub(P.e_pending + e, 1u) - 1u;
            if (left == 0) { // this batch is complete: every trial <= issued has run
                __threadfence();
                uint32_t b = *(volatile uint32_t *)(P.e_best + e);
                uint32_t issued = P.e_issued[e];
                if (b != WF_NONE) wf_finalize_walk(P, w, b, false, s_stats);
                else if (issued >= P.k_max) wf_finalize_walk(P, w, P.k_max, true, s_stats);
                else {
                    uint32_t B = min(2u * P.e_batch[e], P.k_max - issued);
                    P.e_batch[e] = B;
                    P.e_pending[e] = B;
                    P.e_issued[e] = issued + B;
                    __threadfence();
                    if (!wf_push_items(P, e, issued + 1, B)) {
                        // item list full: continue this entry sequentially in this slot
                        P.e_pending[e] = 0;
                        wf_seed(S, g, P, slot, w, issued + 1, F_ITEM | F_SEQ);
                        P.s_entry[slot] = (int32_t)e;
                        wf_append(P, nxt, slot);
                        continue;
                    }
                }
            }
            wf_free(P, slot);
            continue;
        }
        // sequential trials (local, or an entry continued sequentially)
        if (same || trial >= P.k_max) {
            wf_finalize_walk(P, w, trial, !same, s_stats);
            wf_free(P, slot);
            continue;
        }
        if (!item && trial >= WF_LOCAL_TRIALS) {
            unsigned e2 = atomicAdd(&P.hdr->n_entries, 1u);
            if (e2 < P.H) {
                uint32_t B = min(WF_BATCH0, P.k_max - trial);
                P.e_walk[e2] = (int32_t)w;
                P.e_psurf[e2] = psurf;
                P.e_best[e2] = WF_NONE;
                P.e_batch[e2] = B;
                P.e_pending[e2] = B;
                P.e_issued[e2] = trial + B;
                __threadfence();
                if (wf_push_items(P, e2, trial + 1, B)) {
                    wf_free(P, slot);
                    continue;
                }
                P.e_pending[e2] = 0;
            }
        }
        wf_seed(S, g, P, slot, w, trial + 1, fl & (F_ITEM | F_SEQ));
        wf_append(P, nxt, slot);
    }
    // stats
    c_rays = ls.rays;
    atomicAdd(&s_stats[SS_NEWTON], (unsigned long long)c_newton);
    atomicAdd(&s_stats[SS_VTX], (unsigned long long)c_vtx);
    atomicAdd(&s_stats[SS_ATTEMPTS], (unsigned long long)c_att);
    atomicAdd(&s_stats[SS_RAYS], (unsigned long long)c_rays);
    atomicAdd(&s_stats[SS_NODES], (unsigned long long)ls.nodes);
    atomicAdd(&s_stats[SS_TRIS], (unsigned long long)ls.tris);
    __syncthreads();
    if (P.stats)
        for (int j = threadIdx.x; j < SS_N; j += blockDim.x)
            if (s_stats[j]) atomicAdd(P.stats + j, s_stats[j]);
}

// --------------------------------------------------------------------------
// plan (1 thread): snapshot counters, decide the refill assignment and the loop
// --------------------------------------------------------------------------
__global__ void k_wf_plan(const WFParams P) {
    WFHeader *h = P.hdr;
    unsigned par = h->wave & 1u, nxt = par ^ 1u;
    unsigned F = h->free_top;
    unsigned tail = min(h->item_tail, P.C);
    unsigned A = tail > h->item_head ? tail - h->item_head : 0u;
    unsigned long long Q = h->queue < (unsigned long long)P.n ? (unsigned long long)P.n - h->queue : 0ull;
    unsigned a = min(F, A);
    unsigned p = (unsigned)min((unsigned long long)(F - a), Q);
    h->plan_free = F;
    h->plan_items = a;
    h->plan_prims = p;
    h->plan_list = nxt;
    h->plan_queue0 = h->queue;
    h->plan_item0 = h->item_head;
    h->trace_cursor = 0;
    h->item_head += a;
    h->queue += p;
    h->free_top = F - a - p;
    unsigned more = h->list_count[nxt] + a + p;
    // next wave: swap lists, clear the one just consumed
    h->list_count[par] = 0;
    h->wave = h->wave + 1;
    h->more = more;
    if (P.use_cond) cudaGraphSetConditional(P.cond, more > 0 ? 1u : 0u);
}

// --------------------------------------------------------------------------
// refill: free slots <- trial items, then new primary walks
// --------------------------------------------------------------------------
template <int KMAX>
__global__ void k_wf_refill(const DScene S, const SeedCtx g, const WFParams P) {
    const WFHeader *h = P.hdr;
    const unsigned F = h->plan_free, a = h->plan_items, p = h->plan_prims, lst = h->plan_list;
    const unsigned i0 = h->plan_item0;
    const unsigned long long q0 = h->plan_queue0;
    for (unsigned j = blockIdx.x * blockDim.x + threadIdx.x; j < a + p; j += gridDim.x * blockDim.x) {
        uint32_t slot = P.free_stack[F - 1 - j];
        if (j < a) {
            uint32_t e = (uint32_t)P.it_entry[i0 + j];
            uint32_t t = P.it_trial[i0 + j];
            P.s_entry[slot] = (int32_t)e;
            wf_seed(S, g, P, slot, (int64_t)P.e_walk[e], t, F_ITEM);
        } else {
            wf_seed(S, g, P, slot, (int64_t)(q0 + (j - a)), 0u, 0u);
        }
        wf_append(P, lst, slot);
    }
}
