// wavefront.cuh -- wavefront formulation of the batched manifold walk (MPG_FLAG_WAVEFRONT).
//
// The persistent one-chain-per-lane kernel (walk.cuh) runs BVH traversal at
// ~6 active threads per warp (ncu, configs[1]): a lane's next ray depends on
// its own chain, so a warp waits for its slowest traversal and cannot refill
// finished lanes.  Here the walk state lives in S "slots" in global memory
// (SoA) and rays are separated from the chain arithmetic.  One Newton
// iteration of every active slot is one *wave*, run by a CUDA-graph while loop
// (device-side cudaGraphSetConditional, no host round trip):
//
//   for sub-step i = 0 .. KMAX-1:
//     k_wf_rays(i)  pure ray engine over ray list i: persistent warps,
//                   while-while traversal with postponed leaves and dynamic
//                   fetch (a warp refills finished lanes from the list as soon
//                   as fewer than WF_FETCH_MIN lanes are still traversing).
//                   A ray is 32 B (origin, t_max or a hinted triangle, direction, slot | any-hit
//                   bit); a closest hit is written per slot, an any-hit
//                   (visibility) ORs F_FAIL into the slot.
//     k_wf_post(i)  one thread per chain ray of list i: fp64 hit refinement
//                   (R24), surface / type checks (R22, R14), scatter
//                   (deduction, Eq. 6) or next reprojection target (R5), and
//                   emission of ray i+1 into list i+1.
//   k_wf_update     one thread per slot, no traversal: accept/halve (R6),
//                   Newton system fused with block-Thomas (R1-R4, R7), step,
//                   and emission of the next wave's ray 0; at a converged
//                   primary: sides (R8), kappa, G, T (Eq. 2) and its k+1
//                   visibility rays; trials (Eq. 15): sequential up to
//                   WF_LOCAL_TRIALS, then the walk becomes a "hard entry" whose
//                   trials run as independent items in doubling batches; k = the
//                   smallest successful trial (exactly the sequential count).
//   k_wf_plan       one thread: snapshot of free slots / pending items / queue,
//                   assignment plan, counter resets, loop condition.
//   k_wf_refill     assigns trial items, then new primary walks, to free slots
//                   and emits their deduction rays.
//
// Every walk's result depends only on its own counter-based draws, not on the
// slot, lane or wave that ran it: both paths compute the same walks.
#pragma once
#include "walk.cuh"

#define WF_LOCAL_TRIALS 4u
#define WF_BATCH0 4u
#define WF_NONE 0xffffffffu
#define WF_KMAX 8
#ifndef WF_TRACE_MINB
#define WF_TRACE_MINB 8
#endif
#ifndef WF_FETCH_MIN
#define WF_FETCH_MIN 16
#endif
#define WF_ANY (1u << 31)     // ray meta: any-hit over all surfaces (visibility)
// slot flag bits (s_flags); bits 0-15: Newton iteration count
#define F_IT_MASK 0xffffu
#define F_DEDUCE (1u << 16)   // this wave traces the deduction rays
#define F_FAIL (1u << 17)     // a ray of this wave failed (miss / wrong surface / TIR / zero length) or was occluded
#define F_ITEM (1u << 18)     // slot runs a trial item of a hard entry
#define F_SEQ (1u << 20)      // hard entry continued sequentially in this slot (item list full)
#define F_VIS (1u << 21)      // this wave traces the visibility segments of a converged primary

struct WFHeader {                 // device counters (in the workspace; zeroed before k_wf_init)
    unsigned long long queue;     // next primary walk
    unsigned int wave;            // parity of the current slot list / ray list 0
    unsigned int list_count[2];
    unsigned int free_top;        // free-slot stack size
    unsigned int n_entries;       // hard entries published
    unsigned int item_head, item_tail;
    // plan (written by k_wf_plan, read by k_wf_refill)
    unsigned int plan_free, plan_items, plan_prims, plan_list;
    unsigned long long plan_queue0;
    unsigned int plan_item0;
    unsigned int more;            // work remains after this wave (host-loop mode)
    unsigned int ray0_count[2];   // ray list 0, double-buffered by wave parity
    unsigned int ray_count[WF_KMAX];  // ray lists i >= 1
    unsigned int cursor[WF_KMAX];     // ray-engine fetch cursor per sub-step
};

struct WFParams {
    uint32_t trial_base; // Philox trial counter offset of trials t >= 1 (recip_repeats)
    // inputs / outputs (as the persistent kernel)
    const float4 *xD, *nD;
    int64_t n;
    int spp;
    const float4 *seed_xL, *seed_tgt;
    const int *seed_bin;
    const uint32_t *seed_ctype;
    const float *seed_pn;
    uint16_t *out_ctype;
    float4 *chain;
    uint8_t *status;
    uint16_t *iters;
    float *G, *T, *w;
    uint32_t *trials;
    unsigned long long *stats;
    int max_iters, max_iters_long, trials_on;
    uint32_t k_max;
    float tol, beta0, same_eps, ray_eps;
    uint64_t walk_id_base;
    // wavefront state
    WFHeader *hdr;
    uint32_t S;                   // slots
    uint32_t *list[2];
    uint32_t *free_stack;
    // hot per-slot scalars, one 32-B record per slot (one sector per slot access):
    // walk, trial, flags, surf ids of x, surf ids of y, chain type n | bits << 4 |
    // learned << 12 of the current attempt, resolved type string, beta (see rf())
    uint32_t *rec;
    uint32_t *s_psurf;
    uint32_t *s_pct;              // primary chain type n | tau << 4 (trials compare against it)
    float *s_pn;                  // P(n)
    int32_t *s_entry;
    float4 *s_tgt;
    double4 *s_x, *s_y;           // [k][S] chain / traced vertices (fp64 positions, w = prim);
                                  // during deduction s_x[i] holds the fp64 direction of ray i
    double4 *s_dq;                // [k][S] Newton step directions (R: the Newton precision)
    // rays: list 0 double-buffered (S * (KMAX + 1) entries: a chain ray or k+1 visibility rays
    // per slot), lists 1..KMAX-1 (S entries)
    float4 *r0o0, *r0d0, *r0o1, *r0d1;
    float4 *h_p;                  // [S] closest hit point (fp32) | prim (w)
    int32_t *h_s;                 // [S] closest hit surface (-1: miss)
    uint32_t H;                   // hard entry capacity
    int32_t *e_walk;
    uint32_t *e_psurf, *e_pct, *e_best, *e_issued, *e_pending, *e_batch;
    uint32_t C;                   // item capacity
    int32_t *it_entry;
    uint32_t *it_trial;
    cudaGraphConditionalHandle cond;
    int use_cond;                 // 1: inside the CUDA-graph while loop; 0: host-driven waves (profiling)
};

enum { RF_WALK = 0, RF_TRIAL, RF_FLAGS, RF_SURF, RF_YSURF, RF_CTYPE, RF_TAU, RF_BETA };
__device__ __forceinline__ uint32_t &rf(const WFParams &P, uint32_t slot, int f) {
    return P.rec[(size_t)slot * 8 + f];
}
struct SlotRec {   // a whole record, read with two 16-B loads
    uint32_t v[8];
};
__device__ __forceinline__ SlotRec rec_load(const WFParams &P, uint32_t slot) {
    const uint4 *q = reinterpret_cast<const uint4 *>(P.rec + (size_t)slot * 8);
    uint4 a = q[0], b = q[1];
    SlotRec r;
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
    return r;
}

// --------------------------------------------------------------------------
// shared helpers
// --------------------------------------------------------------------------
__device__ __forceinline__ unsigned wf_agg_add(unsigned int *ctr) {   // warp-aggregated atomicAdd(ctr, 1)
    unsigned m = __activemask();
    int leader = __ffs(m) - 1;
    int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(ctr, (unsigned)__popc(m));
    base = __shfl_sync(m, base, leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ void wf_append(const WFParams &P, uint32_t lst, uint32_t slot) {
    P.list[lst][wf_agg_add(&P.hdr->list_count[lst])] = slot;
}

__device__ __forceinline__ void wf_free(const WFParams &P, uint32_t slot) {
    P.free_stack[wf_agg_add(&P.hdr->free_top)] = slot;
    rf(P, slot, RF_WALK) = (uint32_t)(-1);
}

// append a ray to list 0 of wave parity `par`
__device__ __forceinline__ void wf_emit0(const WFParams &P, unsigned par, float3 o, float3 d, float tmax,
                                         uint32_t meta) {
    unsigned idx = wf_agg_add(&P.hdr->ray0_count[par]);
    float4 *ro = par ? P.r0o1 : P.r0o0;
    float4 *rd = par ? P.r0d1 : P.r0d0;
    ro[idx] = make_float4(o.x, o.y, o.z, tmax);
    rd[idx] = make_float4(d.x, d.y, d.z, __uint_as_float(meta));
}

__device__ __forceinline__ double3 ld3(const double4 *a, size_t i) {
    double4 v = a[i];
    return make_double3(v.x, v.y, v.z);
}

// start an attempt (seed) in `slot` for (walk, trial) and emit its deduction ray 0
// into ray list 0 of parity `par` (Eq. 6: x_1 = r(x_D, normalize(target - x_D)))
__device__ __forceinline__ void wf_start(const DScene &S, const SeedCtx &g, const WFParams &P, uint32_t slot,
                                         int64_t w, uint32_t trial, uint32_t extra_flags, unsigned par) {
    float3 tgt = f3(0.f, 0.f, 0.f);
    bool ok;
    uint32_t ct;
    float pn;
    const float3 xD = xyz(__ldg(P.xD + w / P.spp));
    if (trial == 0) {
        ok = __ldg(P.seed_bin + w) != -2;
        tgt = xyz(__ldg(P.seed_tgt + w));
        ct = P.seed_ctype ? __ldg(P.seed_ctype + w) : ((uint32_t)g.k | ((g.tau & 255u) << 4) | (1u << 12));
        pn = P.seed_pn ? __ldg(P.seed_pn + w) : 1.0f;
    } else {
        SeedRes sr;
        ok = seed_target(S, g, P.walk_id_base + w, trial + P.trial_base, xD, xyz(__ldg(P.seed_xL + w)), sr);
        tgt = sr.tgt;
        ct = (uint32_t)sr.n | ((sr.bits & 255u) << 4) | ((sr.learned ? 1u : 0u) << 12);
        pn = sr.Pn;
    }
    rf(P, slot, RF_WALK) = (uint32_t)((int32_t)w);
    rf(P, slot, RF_TRIAL) = trial;
    rf(P, slot, RF_CTYPE) = ct;
    P.s_pn[slot] = pn;
    if (ok) {
        double3 od = d3f(xD);
        double3 v = d3f(tgt) - od;
        double l2 = ddot(v, v);
        ok = l2 > 0.0;
        if (ok) {
            double3 dd = v * rsqrt(l2);
            P.s_x[slot] = make_double4(dd.x, dd.y, dd.z, 0.0);
            wf_emit0(P, par, xD, nrmz(f3d(dd)), __int_as_float(-1), slot);
        }
    }
    rf(P, slot, RF_FLAGS) = F_DEDUCE | extra_flags | (ok ? 0u : F_FAIL);
}

// --------------------------------------------------------------------------
// init: slots 0..min(S,n)-1 <- walks 0..; list[0] = those slots (header zeroed by the host)
// --------------------------------------------------------------------------
template <int KMAX>
__global__ void k_wf_init(const DScene S, const SeedCtx g, const WFParams P) {
    uint32_t s0 = (uint32_t)min((int64_t)P.S, P.n);
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < P.S; s += gridDim.x * blockDim.x) {
        if (s < s0) {
            wf_start(S, g, P, s, (int64_t)s, 0u, 0u, 0u);
            P.list[0][s] = s;
        } else {
            rf(P, s, RF_WALK) = (uint32_t)(-1);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.hdr->queue = s0;
        P.hdr->list_count[0] = s0;
    }
}

// --------------------------------------------------------------------------
// ray engine: closest specular hit (chain rays) or any hit over all surfaces
// (visibility) -- the operator r(x, w) of Eq. 6 and V of Eq. 2.
// Same arithmetic as trace<> in device_common.cuh.
// --------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(128, WF_TRACE_MINB) k_wf_rays(const DScene S, const WFParams P, int sub,
                                                                const float4 *ro_s, const float4 *rd_s) {
    __shared__ unsigned long long s_acc[3];
    if (threadIdx.x < 3) s_acc[threadIdx.x] = 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned par = *(volatile unsigned int *)&P.hdr->wave & 1u;
    const float4 *ro, *rd;
    unsigned count;
    if (sub == 0) {
        ro = par ? P.r0o1 : P.r0o0;
        rd = par ? P.r0d1 : P.r0d0;
        count = *(volatile unsigned int *)&P.hdr->ray0_count[par];
    } else {
        ro = ro_s;
        rd = rd_s;
        count = *(volatile unsigned int *)&P.hdr->ray_count[sub];
    }
    unsigned int *cursor = &P.hdr->cursor[sub];
    const float eps = P.ray_eps;
    const int SENT = 0x7fffffff, NONE = 0;

    int rid = -1;
    bool drained = false;
    uint32_t meta = 0;
    RayW r;
    r.o = r.d = r.idir = f3(0, 0, 0);
    r.kx = r.ky = r.kz = 0;
    r.Sx = r.Sy = r.Sz = 0.f;
    float tmax = 0.f;
    int node = SENT, leaf = NONE, sp = 0;
    int stack[TRAV_STACK(W)];
    int bprim = -2, bsurf = -1;
    float bb0 = 0.f, bb1 = 0.f, bb2 = 0.f;   // barycentrics, or the analytic hit point
    LaneStats ls = {0u, 0u, 0u};

    while (true) {
        // ---- refill finished lanes (one atomic per warp) ----
        unsigned im = __ballot_sync(MPG_FULL, rid < 0 && !drained);
        if (im) {
            int leader = __ffs(im) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(cursor, (unsigned)__popc(im));
            base = __shfl_sync(MPG_FULL, base, leader);
            if (rid < 0 && !drained) {
                unsigned idx = base + __popc(im & ((1u << lane) - 1u));
                if (idx < count) {
                    rid = (int)idx;
                    float4 a = ro[idx], b = rd[idx];
                    float3 o = xyz(a), d = xyz(b);
                    meta = __float_as_uint(b.w);
                    const bool any = (meta & WF_ANY) != 0;
                    // any-hit rays carry t_max; chain rays a hinted triangle (or -1), t_max = inf
                    tmax = any ? a.w : 3.0e38f;
                    const int hint = any ? -1 : __float_as_int(a.w);
                    ls.rays++;
                    bsurf = -1;
                    bprim = -2;
                    for (int s = 0; s < S.n_surf; s++) {
                        const DSurf &f = S.surf[s];
                        if (f.kind == 2 || (!any && f.mat == 2)) continue;
                        float t;
                        float3 p;
                        bool hit;
                        if (f.kind == 0) hit = sphere_hit(o, d, f.center, f.radius, eps, tmax, t, p);
                        else {
                            hit = quad_hit(o, d, f.origin, f.eu, f.ev, eps, tmax, t);
                            p = o + d * t;
                        }
                        if (hit) { tmax = t; bsurf = s; bprim = -1; bb0 = p.x; bb1 = p.y; bb2 = p.z; }
                    }
                    node = SENT;
                    leaf = NONE;
                    if (S.n_tri > 0 && !(any && bsurf >= 0)) {
                        ray_setup(r, o, d);
                        if (hint >= 0) { // bound the search by the hinted triangle (see trace<>)
                            ls.tris++;
                            float4 p0 = __ldg(S.tpos + TSTRIDE * hint), p1 = __ldg(S.tpos + TSTRIDE * hint + 1),
                                   p2 = __ldg(S.tpos + TSTRIDE * hint + 2);
                            float t, c0, c1, c2;
                            if (__float_as_int(p2.w) != 0 &&
                                tri_hit(r, xyz(p0), xyz(p1), xyz(p2), eps, tmax, t, c0, c1, c2)) {
                                tmax = t; bprim = hint; bsurf = __float_as_int(p1.w);
                                bb0 = c0; bb1 = c1; bb2 = c2;
                            }
                        }
                        node = 0;
                        stack[0] = SENT;
                        sp = 1;
                    }
                } else {
                    drained = true;
                }
            }
        }
        if (__all_sync(MPG_FULL, rid < 0)) break;

        // ---- traverse until done, or until the warp is too sparse (dynamic fetch) ----
        if (rid >= 0) {
            const bool any = (meta & WF_ANY) != 0;
            const float3 o = r.o;
            const float3 oi = f3(o.x * r.idir.x, o.y * r.idir.y, o.z * r.idir.z);
            while (node != SENT || leaf != NONE) {
                while (node >= 0 && node != SENT) {
                    ls.nodes++;
                    node = bvh_visit<W>(S.nodes, node, oi, r.idir, eps, tmax, stack, sp);
                    if (node < 0 && leaf == NONE) { // postpone the leaf, keep traversing
                        leaf = node;
                        node = stack[--sp];
                    }
                    if (!__any_sync(__activemask(), leaf == NONE)) break;
                }
                while (leaf != NONE) {
                    int v = ~leaf;
                    int start = v >> 3, cnt = (v & 7) + 1;
                    bool found = false;
                    for (int j = start; j < start + cnt; j++) {
                        ls.tris++;
                        float4 p0 = __ldg(S.tpos + TSTRIDE * j), p1 = __ldg(S.tpos + TSTRIDE * j + 1),
                               p2 = __ldg(S.tpos + TSTRIDE * j + 2);
                        if (!any && __float_as_int(p2.w) == 0) continue;
                        float t, c0, c1, c2;
                        if (tri_hit(r, xyz(p0), xyz(p1), xyz(p2), eps, tmax, t, c0, c1, c2)) {
                            tmax = t; bprim = j; bsurf = __float_as_int(p1.w);
                            bb0 = c0; bb1 = c1; bb2 = c2;
                            if (any) { found = true; break; }
                        }
                    }
                    if (found) { node = SENT; leaf = NONE; break; }
                    leaf = NONE;
                    if (node < 0) { // the traversal stopped on another leaf
                        leaf = node;
                        node = stack[--sp];
                    }
                }
                if (__popc(__activemask()) < WF_FETCH_MIN) break;
            }
            if (node == SENT && leaf == NONE) { // ray done
                const uint32_t slot = meta & ~WF_ANY;
                if (any) {
                    if (bsurf >= 0) atomicOr(&rf(P, slot, RF_FLAGS), F_FAIL);
                } else {
                    float3 pf;
                    if (bprim >= 0) {
                        float3 v0 = xyz(__ldg(S.tpos + TSTRIDE * bprim)), v1 = xyz(__ldg(S.tpos + TSTRIDE * bprim + 1)),
                               v2 = xyz(__ldg(S.tpos + TSTRIDE * bprim + 2));
                        pf = v0 * bb0 + v1 * bb1 + v2 * bb2;
                    } else {
                        pf = f3(bb0, bb1, bb2);
                    }
                    P.h_p[slot] = make_float4(pf.x, pf.y, pf.z, __int_as_float(bprim));
                    P.h_s[slot] = bsurf;
                }
                rid = -1;
            }
        }
    }
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
// post: vertex i of every chain ray of list i -- refine, check, emit ray i+1
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_wf_post(const DScene S, const WFParams P, int sub, const float4 *rd_s,
                                                 float4 *ro_n, float4 *rd_n) {
    const unsigned par = *(volatile unsigned int *)&P.hdr->wave & 1u;
    const float4 *rd = sub == 0 ? (par ? P.r0d1 : P.r0d0) : rd_s;
    const unsigned count = sub == 0 ? *(volatile unsigned int *)&P.hdr->ray0_count[par]
                                    : *(volatile unsigned int *)&P.hdr->ray_count[sub];
    const int i = sub;
    for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < count; idx += gridDim.x * blockDim.x) {
        const uint32_t meta = __float_as_uint(rd[idx].w);
        if (meta & WF_ANY) continue;
        const uint32_t slot = meta;
        const SlotRec SR = rec_load(P, slot);
        const uint32_t fl = SR.v[RF_FLAGS];
        const bool ded = (fl & F_DEDUCE) != 0;
        const int hs = P.h_s[slot];
        const float4 hp = P.h_p[slot];
        const int prim = __float_as_int(hp.w);
        const uint32_t ct = SR.v[RF_CTYPE];
        const int k = (int)(ct & 15u);
        bool ok = hs >= 0 && (ded || hs == (int)((SR.v[RF_SURF] >> (4 * i)) & 15u));
        uint32_t bit = 0;
        if (ok && ded) { // resolve the type of vertex i (R22, R14)
            bit = (ct >> (4 + i)) & 1u;
            const int mat = S.surf[hs].mat;
            if (!((ct >> 12) & 1u) && mat == 0) bit = 0u;
            if (bit && mat != 1) ok = false;
        }
        if (!ok) {
            rf(P, slot, RF_FLAGS) = fl | F_FAIL;
            continue;
        }
        const int64_t wk = (int32_t)SR.v[RF_WALK];
        const double3 od = i == 0 ? d3f(xyz(__ldg(P.xD + wk / P.spp))) : ld3(P.s_y, (size_t)(i - 1) * P.S + slot);
        double3 tg;
        const double bt = (double)__uint_as_float(SR.v[RF_BETA]);
        if (ded) tg = od + ld3(P.s_x, (size_t)i * P.S + slot);
        else {
            double4 x4 = P.s_x[(size_t)i * P.S + slot];
            double4 dq4 = P.s_dq[(size_t)i * P.S + slot];
            tg = make_double3(x4.x + dq4.x * bt, x4.y + dq4.y * bt, x4.z + dq4.z * bt);
        }
        // the hit on the exact line, in fp64 (R24)
        const double3 y = refine_hit(S, prim, hs, od, tg, xyz(hp));
        P.s_y[(size_t)i * P.S + slot] = make_double4(y.x, y.y, y.z, (double)prim);
        rf(P, slot, RF_YSURF) = (i == 0 ? 0u : SR.v[RF_YSURF]) | ((uint32_t)(hs & 15) << (4 * i));
        if (ded) rf(P, slot, RF_TAU) = (i == 0 ? 0u : SR.v[RF_TAU]) | (bit << i);
        if (i + 1 < k) { // ray i+1 from y_i
            double3 dd;
            if (ded) {
                dd = ld3(P.s_x, (size_t)i * P.S + slot);
                if (!scatter_dir(S, dd, prim, hs, f3d(y), bit)) {
                    rf(P, slot, RF_FLAGS) = fl | F_FAIL;
                    continue;
                }
                P.s_x[(size_t)(i + 1) * P.S + slot] = make_double4(dd.x, dd.y, dd.z, 0.0);
            } else {
                double4 x4 = P.s_x[(size_t)(i + 1) * P.S + slot];
                double4 dq4 = P.s_dq[(size_t)(i + 1) * P.S + slot];
                double3 q = make_double3(x4.x + dq4.x * bt, x4.y + dq4.y * bt, x4.z + dq4.z * bt);
                double3 v = q - y;
                double l2 = ddot(v, v);
                if (!(l2 > 0.0)) {
                    rf(P, slot, RF_FLAGS) = fl | F_FAIL;
                    continue;
                }
                dd = v * rsqrt(l2);
            }
            const int hint = ded ? -1 : (int)P.s_x[(size_t)(i + 1) * P.S + slot].w;
            unsigned j = wf_agg_add(&P.hdr->ray_count[i + 1]);
            float3 o = f3d(y), d = nrmz(f3d(dd));
            ro_n[j] = make_float4(o.x, o.y, o.z, __int_as_float(hint));
            rd_n[j] = make_float4(d.x, d.y, d.z, __uint_as_float(slot));
        }
    }
}

// --------------------------------------------------------------------------
// hard entries: finalize / next batch
// --------------------------------------------------------------------------
__device__ __forceinline__ void wf_finalize_walk(const WFParams &P, int64_t w, uint32_t kk, bool truncated,
                                                 unsigned long long *s_stats) {
    P.trials[w] = kk;
    float pn = P.seed_pn ? __ldg(P.seed_pn + w) : 1.0f;
    P.w[w] = P.T[w] * (float)kk / (pn * __ldg(P.seed_xL + w).w);
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

__device__ __forceinline__ void wf_primary_status(const WFParams &P, int64_t w, int st, int it,
                                                  unsigned long long *s_stats) {
    P.status[w] = (uint8_t)st;
    P.iters[w] = (uint16_t)it;
    atomicAdd(&s_stats[SS_STATUS0 + st], 1ull);
    atomicAdd(&s_stats[SS_PRIM_IT], (unsigned long long)it);
    atomicAdd(&s_stats[SS_WALKS], 1ull);
    if (st == ST_CONVERGED || st == ST_OCCLUDED) atomicAdd(&s_stats[SS_CONV], 1ull);
}

// --------------------------------------------------------------------------
// update: one thread per slot of this wave (no traversal)
// --------------------------------------------------------------------------
template <int KMAX, typename R>
__global__ void __launch_bounds__(128, 4) k_wf_update(const DScene S, const SeedCtx g, const WFParams P) {
    __shared__ unsigned long long s_stats[SS_N];
    for (int j = threadIdx.x; j < SS_N; j += blockDim.x) s_stats[j] = 0ull;
    __syncthreads();
    const unsigned par = *(volatile unsigned int *)&P.hdr->wave & 1u;
    const uint32_t *list = P.list[par];
    const unsigned count = *(volatile unsigned int *)&P.hdr->list_count[par];
    const unsigned nxt = par ^ 1u;
    uint32_t c_newton = 0, c_vtx = 0, c_att = 0;

    for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < count; idx += gridDim.x * blockDim.x) {
        const uint32_t slot = list[idx];
        const SlotRec SR = rec_load(P, slot);
        const uint32_t fl = SR.v[RF_FLAGS];
        const int64_t w = (int32_t)SR.v[RF_WALK];
        const uint32_t trial = SR.v[RF_TRIAL];
        int it = (int)(fl & F_IT_MASK);
        const uint32_t ct = SR.v[RF_CTYPE];
        const int k = max(1, min((int)(ct & 15u), KMAX));

        // ---------------- visibility result of a converged primary ----------------
        if (fl & F_VIS) {
            const bool occluded = (fl & F_FAIL) != 0;
            float Tv = P.T[w];
            if (occluded) { P.G[w] = 0.f; P.T[w] = 0.f; Tv = 0.f; }
            wf_primary_status(P, w, occluded ? ST_OCCLUDED : ST_CONVERGED, it, s_stats);
            if (!occluded && Tv > 0.0f && P.trials_on) {
                wf_start(S, g, P, slot, w, 1u, 0u, nxt);
                wf_append(P, nxt, slot);
            } else {
                P.trials[w] = 0;
                P.w[w] = 0.0f;
                wf_free(P, slot);
            }
            continue;
        }

        float beta = __uint_as_float(SR.v[RF_BETA]);
        const bool deduce = fl & F_DEDUCE, failed = fl & F_FAIL;
        const uint32_t tau = SR.v[RF_TAU];
        double3 x[KMAX];
        V3<R> sg[KMAX], tg[KMAX], dq[KMAX];
        int prim[KMAX], surf[KMAX];
        R Di[KMAX][4], Ub[KMAX][4];
        const uint32_t sp_ = failed ? SR.v[RF_SURF] : SR.v[RF_YSURF];
        const double4 *src = failed ? P.s_x : P.s_y;
#pragma unroll
        for (int j = 0; j < KMAX; j++) {
            sg[j] = tg[j] = dq[j] = mk3<R>(0, 0, 0);
            if (j >= k) { x[j] = make_double3(0, 0, 0); prim[j] = -1; surf[j] = 0; continue; }
            double4 v = src[(size_t)j * P.S + slot];
            x[j] = make_double3(v.x, v.y, v.z);
            prim[j] = (int)v.w;
            surf[j] = (int)((sp_ >> (4 * j)) & 15u);
        }
        int end = -1;
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
        const float3 xL = xyz(__ldg(P.seed_xL + w));
        bool singular = false;
        if (end < 0) {
            if (fresh) {
                c_vtx += k;
                float cm;
                int rr = newton_system<KMAX, R>(S, k, tau, xD, xL, x, prim, surf, P.tol, Di, Ub, sg, tg, dq,
                                                    singular, cm);
                if (rr == 1) end = ST_CONVERGED;
                else if (rr == 2) end = ST_DEGENERATE;
                else {
#pragma unroll
                    for (int j = 0; j < KMAX; j++)
                        if (j < k) P.s_dq[(size_t)j * P.S + slot] = make_double4(dq[j].x, dq[j].y, dq[j].z, 0.0);
                }
            }
            if (end < 0 && it >= ((k >= 3 && P.max_iters_long > 0) ? P.max_iters_long : P.max_iters)) end = ST_MAXITER;
        }
        if (fresh) {
#pragma unroll
            for (int j = 0; j < KMAX; j++)
                if (j < k) P.s_x[(size_t)j * P.S + slot] = make_double4(x[j].x, x[j].y, x[j].z, (double)prim[j]);
            rf(P, slot, RF_SURF) = sp_;
        }
        if (end < 0) { // continue: reprojection ray 0 toward q_0 = x_0 + beta dq_0 next wave (R5)
            rf(P, slot, RF_BETA) = __float_as_uint(beta);
            double3 d0;
            if (fresh) d0 = make_double3((double)dq[0].x, (double)dq[0].y, (double)dq[0].z);
            else d0 = ld3(P.s_dq, slot);
            const double bt = (double)beta;
            double3 q = make_double3(x[0].x + d0.x * bt, x[0].y + d0.y * bt, x[0].z + d0.z * bt);
            double3 v = q - d3f(xD);
            double l2 = ddot(v, v);
            bool ok = l2 > 0.0;
            if (ok) wf_emit0(P, nxt, xD, nrmz(f3d(v * rsqrt(l2))), __int_as_float(prim[0]), slot);
            rf(P, slot, RF_FLAGS) = (fl & (F_ITEM | F_SEQ)) | (uint32_t)it | (ok ? 0u : F_FAIL);
            wf_append(P, nxt, slot);
            continue;
        }
        // ---------------- attempt ended ----------------
        c_newton += it;
        c_att++;
        int lid = 0;
        if (S.n_light > 1) lid = (int)uidx(rng_draw(g.seed, P.walk_id_base + w, 0u, 0u).z, (uint32_t)S.n_light);
        if (trial == 0) {
            int st = end;
            float Gv = 0.f, Tv = 0.f;
            if (st == ST_CONVERGED) {
                const DLight &L = S.light[lid];
                float kap;
                R DL[4];
                if (!post_sweep<KMAX, R>(S, L, k, tau, xD, xL, x, prim, surf, true, kap, DL)) st = ST_BAD_SIDE;
                else {
                    Gv = singular ? 0.0f : ggt_from_blocks<KMAX, R>(k, xD, xyz(__ldg(P.nD + w / P.spp)), x, Di,
                                                                        Ub, sg, tg, DL);
                    float Le = L.emit;
                    if (L.kind == 1 && !(dot(f3d(x[k - 1]) - xL, L.n) > 0.0f)) Le = 0.0f;
                    Tv = kap * Gv * Le;
                }
            }
            if (st != ST_SEED_FAIL) {
#pragma unroll
                for (int j = 0; j < KMAX; j++) {
                    if (j >= k) break;
                    int pid = prim[j] >= 0 ? __float_as_int(__ldg(S.tpos + TSTRIDE * prim[j]).w) : -1;
                    P.chain[(int64_t)j * P.n + w] = make_float4((float)x[j].x, (float)x[j].y, (float)x[j].z,
                                                                __int_as_float(pid));
                }
            }
            P.G[w] = Gv;
            P.T[w] = Tv;
            if (P.out_ctype) P.out_ctype[w] = (uint16_t)((uint32_t)k | (tau << 4));
            if (st == ST_CONVERGED) { // the k+1 visibility segments are traced next wave
                P.s_psurf[slot] = sp_;
                P.s_pct[slot] = (uint32_t)k | (tau << 4);
                rf(P, slot, RF_FLAGS) = F_VIS | (uint32_t)it;
                float3 a = xD;
#pragma unroll 1
                for (int j = 0; j <= k; j++) { // fp32 segments as walk.cuh
                    float3 bq = j == k ? xL : f3d(x[j]);
                    float3 dv = bq - a;
                    float l = len(dv);
                    wf_emit0(P, nxt, a, dv * (1.0f / l), l - P.ray_eps, slot | WF_ANY);
                    a = bq;
                }
                wf_append(P, nxt, slot);
            } else {
                wf_primary_status(P, w, st, it, s_stats);
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
        const uint32_t pct = item ? P.e_pct[e] : P.s_pct[slot];
        bool same = false;
        if (end == ST_CONVERGED && (uint32_t)k == (pct & 15u) && tau == (pct >> 4)) {
            float kd;
            R DLd[4];
            if (post_sweep<KMAX, R>(S, S.light[lid], k, tau, xD, xL, x, prim, surf, false, kd, DLd)) {
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
                        wf_start(S, g, P, slot, w, issued + 1, F_ITEM | F_SEQ, nxt);
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
                P.e_pct[e2] = pct;
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
        wf_start(S, g, P, slot, w, trial + 1, fl & (F_ITEM | F_SEQ), nxt);
        if (item) P.s_entry[slot] = (int32_t)e;
        wf_append(P, nxt, slot);
    }
    // warp-reduce the per-thread counters: one shared atomic per warp and counter
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        c_newton += __shfl_down_sync(MPG_FULL, c_newton, off);
        c_vtx += __shfl_down_sync(MPG_FULL, c_vtx, off);
        c_att += __shfl_down_sync(MPG_FULL, c_att, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c_newton) atomicAdd(&s_stats[SS_NEWTON], (unsigned long long)c_newton);
        if (c_vtx) atomicAdd(&s_stats[SS_VTX], (unsigned long long)c_vtx);
        if (c_att) atomicAdd(&s_stats[SS_ATTEMPTS], (unsigned long long)c_att);
    }
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
    h->item_head += a;
    h->queue += p;
    h->free_top = F - a - p;
    unsigned more = h->list_count[nxt] + a + p;
    h->list_count[par] = 0;   // next wave: swap lists, clear the ones just consumed
    h->ray0_count[par] = 0;
    for (int i = 0; i < WF_KMAX; i++) {
        h->ray_count[i] = 0;
        h->cursor[i] = 0;
    }
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
            wf_start(S, g, P, slot, (int64_t)P.e_walk[e], t, F_ITEM, lst);
        } else {
            wf_start(S, g, P, slot, (int64_t)(q0 + (j - a)), 0u, 0u, lst);
        }
        wf_append(P, lst, slot);
    }
}
