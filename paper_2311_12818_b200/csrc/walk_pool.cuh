// walk_pool.cuh -- the warp-specialized manifold-walk kernel (sm_100a), round 2.
//
// Same method and same per-walk arithmetic as walk.cuh (it calls the same device
// functions: trace<W>, refine_hit, scatter_dir, newton_system, post_sweep,
// ggt_from_blocks, seed_target and the trial bookkeeping), different execution model.
//
// walk.cuh binds one walk to one lane for the walk's whole life, so a warp
// instruction of the traversal, of the Newton sweep or of the end-of-attempt logic
// runs on the 8-12 lanes that happen to be in that phase (ncu), all
// phases share one register budget (64: ~1 KB of spills per lane, 0.5 TB of
// local-memory DRAM traffic per configs[2] launch) and every warp walks through the
// whole 60 KB of code (41 % instruction-fetch stalls).
//
// Here a block (one per SM) owns a pool of NV walk *slots* whose state lives in
// shared memory, and its warps are specialized:
//   * trace warps pop slots that need rays from the ray queue and run only the
//     chain-ray loop (deduction, reprojection with its step-halving retries, or the
//     k+1 visibility segments): every lane with a slot traces a ray in every
//     iteration, finished lanes refill from the queue at once (north_star's
//     "compaction to regroup still-iterating chains"), few registers;
//   * compute warps pop slots with a fresh chain from the solve queue and run the
//     Newton sweep on 32 of them at once (many registers: setmaxnreg hands them the
//     trace warps' surplus), and pop slots whose attempt ended from the control queue
//     (end-of-attempt bookkeeping, reciprocal-probability trials, fetch of the next
//     primary, trial seeds), or poll the trial-item ring for slots that wait.
// Queues are rings of slot ids in shared memory.  The global work distribution
// (primary queue, hard entries, trial items by ticket, `resolved` count) is
// walk.cuh's, with a slot in the place of a lane, so the trial count k of every walk
// is the same sequential count (Eq. 15, R13) and outputs are bit-identical.
#pragma once
#include "walk.cuh"

enum { PQ_RAY = 0, PQ_HIT = 1, PQ_SOLVE = 2, PQ_CTL = 3, PQ_WAIT = 4, PQ_N = 5 };
enum { PS_TRACE = 0, PS_HIT = 1, PS_SOLVE = 2, PS_CTL = 3, PS_SLEEP = 4, PS_EXIT = 5 };

// MPG_POOL_PROF: diagnostic build (tools/pool_prof.py): per-role cycle and batch counters
#ifdef MPG_POOL_PROF
// per warp: 0 R phases, 12 H phases, 1 S phases, 4 C phases, 2 R cycles, 3 H cycles, 7 S cycles, 10 C cycles,
// 11 scheduler + barrier cycles, 5 solve batches, 6 solve slots, 8 control batches, 9 control slots
__device__ unsigned long long g_pool_prof[16];
#define PROF_DECL unsigned long long pf_[16] = {0}; long long pf_t = clock64();
#define PROF_ADD(i, v) (pf_[i] += (unsigned long long)(v))
#define PROF_LAP(i) { const long long t_ = clock64(); pf_[i] += (unsigned long long)(t_ - pf_t); pf_t = t_; }
#define PROF_FLUSH if (lane == 0) { for (int i_ = 0; i_ < 16; i_++) if (pf_[i_]) atomicAdd(&g_pool_prof[i_], pf_[i_]); }
#else
#define PROF_DECL
#define PROF_ADD(i, v)
#define PROF_LAP(i)
#define PROF_FLUSH
#endif

struct PoolShared {
    unsigned head[PQ_N], tail[PQ_N];
    unsigned end[PQ_N];     // phase snapshot of the tails (entries present when the phase began)
    unsigned sel;           // phase chosen by the scheduler thread
    unsigned progress;      // a control phase moved some slot on
    unsigned done, drained;
    unsigned stats[SS_N];
};

// slot word `st`: it (16) | end_status (3) << 16 | occluded << 19 | seq_only << 20 | phase (4) << 24 | lid (3) << 28
// slot word `ct`: k (4) | tau (8) << 4 | bits (8) << 12 | learned << 20 | cur << 21 | ti (3) << 22
// (tau holds the types resolved so far while a deduction is being traced; ti = the chain ray in flight)
#define ST_IT(s) ((int)((s)&0xffffu))
#define ST_END(s) ((int)(((s) >> 16) & 7u))
#define ST_OCC(s) ((((s) >> 19) & 1u) != 0u)
#define ST_SEQ(s) ((((s) >> 20) & 1u) != 0u)
#define ST_PH(s) ((int)(((s) >> 24) & 15u))
#define ST_LID(s) ((int)(((s) >> 28) & 7u))
__device__ __forceinline__ uint32_t st_pack(int it, int end_status, bool occ, bool seq, int phase, int lid) {
    return (uint32_t)(it & 0xffff) | ((uint32_t)(end_status & 7) << 16) | ((occ ? 1u : 0u) << 19) |
           ((seq ? 1u : 0u) << 20) | ((uint32_t)(phase & 15) << 24) | ((uint32_t)(lid & 7) << 28);
}
__device__ __forceinline__ uint32_t ct_pack(int k, uint32_t tau, uint32_t bits, bool learned, int cur, int ti = 0) {
    return (uint32_t)(k & 15) | ((tau & 255u) << 4) | ((bits & 255u) << 12) | ((learned ? 1u : 0u) << 20) |
           ((uint32_t)(cur & 1) << 21) | ((uint32_t)(ti & 7) << 22);
}
#define CT_TI(c) ((int)(((c) >> 22) & 7u))

template <int KMAX, typename R> struct Pool {
    int nv, nvq;
    double *xb;            // [2][KMAX][3][nv] chain vertices: buffer cur = the chain, cur^1 = the chain being traced
    R *dq;                 // [KMAX][3][nv] Newton step (world space); [0] doubles as the seed target during deduction
    int *pr;               // [2][KMAX][nv] primitives
    uint32_t *sf;          // [2][nv] surface ids, 4 bits per vertex
    uint32_t *w, *trial, *ct, *pct, *psurf, *st, *ticket;
    int *item_e;
    float *beta, *Tprim, *Gc, *Tc, *xD;   // xD [3][nv]
    float *ray;            // [8][nv] the ray in flight: o, d, tmax, hint (-1 none, -2 any-hit over all surfaces);
                           // then its hit: point, -, -, -, surface, primitive (-1 analytic, -3 miss, <= -16 no ray: -16 - code)
    unsigned short *ring;  // [PQ_N][nvq] slot + 1 (0: empty)
    static __host__ __device__ size_t slot_bytes() {
        return (size_t)KMAX * (48 + 3 * sizeof(R) + 8) + 8 + 7 * 4 + 4 + 4 * 4 + 12 + 32;
    }
    static __host__ __device__ size_t bytes(int nv, int nvq) { return slot_bytes() * nv + (size_t)PQ_N * nvq * 2 + 64; }
    // slot arrays at `base`, queue rings at `rings` (shared memory)
    __device__ void carve(unsigned char *base, unsigned char *rings, int nv_, int nvq_) {
        nv = nv_; nvq = nvq_;
        unsigned char *p = base;
        xb = (double *)p; p += (size_t)2 * KMAX * 3 * nv * 8;
        dq = (R *)p; p += (size_t)KMAX * 3 * nv * sizeof(R);
        pr = (int *)p; p += (size_t)2 * KMAX * nv * 4;
        sf = (uint32_t *)p; p += (size_t)2 * nv * 4;
        w = (uint32_t *)p; p += (size_t)nv * 4;
        trial = (uint32_t *)p; p += (size_t)nv * 4;
        ct = (uint32_t *)p; p += (size_t)nv * 4;
        pct = (uint32_t *)p; p += (size_t)nv * 4;
        psurf = (uint32_t *)p; p += (size_t)nv * 4;
        st = (uint32_t *)p; p += (size_t)nv * 4;
        ticket = (uint32_t *)p; p += (size_t)nv * 4;
        item_e = (int *)p; p += (size_t)nv * 4;
        beta = (float *)p; p += (size_t)nv * 4;
        Tprim = (float *)p; p += (size_t)nv * 4;
        Gc = (float *)p; p += (size_t)nv * 4;
        Tc = (float *)p; p += (size_t)nv * 4;
        xD = (float *)p; p += (size_t)3 * nv * 4;
        ray = (float *)p; p += (size_t)8 * nv * 4;
        ring = rings ? (unsigned short *)rings : (unsigned short *)p;
    }
    __device__ __forceinline__ double3 getx(int buf, int i, int s) const {
        const double *p = xb + (size_t)((buf * KMAX + i) * 3) * nv + s;
        return make_double3(p[0], p[nv], p[2 * nv]);
    }
    __device__ __forceinline__ void setx(int buf, int i, int s, double3 v) {
        double *p = xb + (size_t)((buf * KMAX + i) * 3) * nv + s;
        p[0] = v.x; p[nv] = v.y; p[2 * nv] = v.z;
    }
    __device__ __forceinline__ V3<R> getdq(int i, int s) const {
        const R *p = dq + (size_t)(i * 3) * nv + s;
        return mk3<R>(p[0], p[nv], p[2 * nv]);
    }
    __device__ __forceinline__ void setdq(int i, int s, V3<R> v) {
        R *p = dq + (size_t)(i * 3) * nv + s;
        p[0] = v.x; p[nv] = v.y; p[2 * nv] = v.z;
    }
    __device__ __forceinline__ void set_ray(int s, float3 o, float3 d, float tmax, int hint) {
        ray[s] = o.x; ray[nv + s] = o.y; ray[2 * nv + s] = o.z;
        ray[3 * nv + s] = d.x; ray[4 * nv + s] = d.y; ray[5 * nv + s] = d.z;
        ray[6 * nv + s] = tmax; ray[7 * nv + s] = __int_as_float(hint);
    }
    // no ray could be formed (zero length, failed scatter): the pass ends with `code` in the hit phase
    __device__ __forceinline__ void set_noray(int s, int code) { ray[7 * nv + s] = __int_as_float(-16 - code); }
    __device__ __forceinline__ void set_hit(int s, float3 p, int surf, int prim) {
        ray[s] = p.x; ray[nv + s] = p.y; ray[2 * nv + s] = p.z;
        ray[6 * nv + s] = __int_as_float(surf); ray[7 * nv + s] = __int_as_float(prim);
    }
    __device__ __forceinline__ float3 getxD(int s) const { return f3(xD[s], xD[nv + s], xD[2 * nv + s]); }
    __device__ __forceinline__ void setxD(int s, float3 v) { xD[s] = v.x; xD[nv + s] = v.y; xD[2 * nv + s] = v.z; }
    __device__ __forceinline__ int getpr(int buf, int i, int s) const { return pr[(size_t)(buf * KMAX + i) * nv + s]; }
    __device__ __forceinline__ void setpr(int buf, int i, int s, int v) { pr[(size_t)(buf * KMAX + i) * nv + s] = v; }
};

// ---- queues: rings of slot ids; a slot is in at most one queue, so a ring of >= nv entries never
// overflows.  Producers reserve positions with one atomicAdd per warp and then write the entries;
// consumers reserve [head, head + take) below the reserved tail with a CAS and wait (briefly: the
// producer is between its atomicAdd and its store) for each entry to appear.
// (one atomicAdd per reservation; a reservation that reaches past `end` is cut there and the
// overshoot of `head` is undone by the scheduler thread after the phase, when no one reserves)
__device__ __forceinline__ int q_reserve(PoolShared *sh, int q, int want, unsigned &base, unsigned end) {
    if ((int)(end - *(volatile unsigned *)&sh->head[q]) <= 0) return 0;
    base = atomicAdd(&sh->head[q], (unsigned)want);
    return max(0, min(want, (int)(end - base)));
}
__device__ __forceinline__ unsigned q_tail(PoolShared *sh, int q) { return *(volatile unsigned *)&sh->tail[q]; }
template <int KMAX, typename R>
__device__ __forceinline__ int q_take(const Pool<KMAX, R> &pl, int q, unsigned pos) {
    volatile unsigned short *e = pl.ring + (size_t)q * pl.nvq + (pos & (unsigned)(pl.nvq - 1));
    unsigned short v;
    while ((v = *e) == 0) {}
    *e = 0;
    __threadfence_block();
    return (int)v - 1;
}
// push the slots of the lanes with `flag` (whole warp calls it)
template <int KMAX, typename R>
__device__ __forceinline__ void q_push(const Pool<KMAX, R> &pl, PoolShared *sh, int q, bool flag, int slot, int lane) {
    const unsigned m = __ballot_sync(MPG_FULL, flag);
    if (!m) return;
    const int leader = __ffs(m) - 1;
    unsigned base = 0;
    __threadfence_block();   // the slot's state before its id
    if (lane == leader) base = atomicAdd(&sh->tail[q], (unsigned)__popc(m));
    base = __shfl_sync(MPG_FULL, base, leader);
    if (flag) {
        const unsigned pos = base + (unsigned)__popc(m & ((1u << lane) - 1u));
        volatile unsigned short *e = pl.ring + (size_t)q * pl.nvq + (pos & (unsigned)(pl.nvq - 1));
        while (*e != 0) {}   // the consumer of the previous lap is clearing it
        *e = (unsigned short)(slot + 1);
    }
    __syncwarp();
}

// ============================================================================
// ray phase: nothing but BVH traversal.  A lane takes the ray of a slot from the ray queue,
// traverses, writes the hit into the slot and hands the slot to the hit queue.  Lanes whose
// ray ends take the next one as soon as `refill` lanes of the warp are idle (persistent
// while-while traversal with dynamic fetch, Aila & Laine 2009), so the traversal loop runs
// on nearly full warps although ray lengths differ widely.  Same closest / any hit as
// trace<W> (device_common.cuh): same node order, same tests, same tie rules.
// ============================================================================
template <int KMAX, typename R, int W>
__device__ __forceinline__ void pool_ray_phase(const DScene &S, const WalkParams &P, Pool<KMAX, R> &pl, PoolShared *sh,
                                               const int lane, const unsigned r_end, const int refill,
                                               unsigned long long &rays, LaneStats &st) {
    const int SENT = 0x7fffffff, NONE = 0;
    const float eps = P.ray_eps;
    int slot = -1;
    bool active = false, fin = false, more = true;
    bool any = false, spec_only = true;
    float best = 0.f, bb0 = 0.f, bb1 = 0.f, bb2 = 0.f;
    int bprim = -2, bsurf = -1;
    float3 bp = f3(0.f, 0.f, 0.f), oi = f3(0.f, 0.f, 0.f);
    RayW r;
    r.o = r.d = r.idir = f3(0.f, 0.f, 1.f);
    r.kx = 0; r.ky = 1; r.kz = 2; r.Sx = r.Sy = 0.f; r.Sz = 1.f;
    int stack[TRAV_STACK(W)];
    int sp = 1, node = SENT, leaf = NONE;
    while (true) {
        // ---- finished rays: the hit goes to the slot, the slot to the hit queue --------------
        if (fin) {
            float3 hp = bp;
            int hprim = bprim;
            if (bsurf < 0) hprim = -3;
            else if (bprim >= 0 && !any) {
                const float3 v0 = xyz(__ldg(S.tpos + TSTRIDE * bprim)), v1 = xyz(__ldg(S.tpos + TSTRIDE * bprim + 1)),
                             v2 = xyz(__ldg(S.tpos + TSTRIDE * bprim + 2));
                hp = v0 * bb0 + v1 * bb1 + v2 * bb2;
            }
            pl.set_hit(slot, hp, bsurf, hprim);
        }
        q_push(pl, sh, PQ_HIT, fin, slot, lane);
        if (fin) { fin = false; slot = -1; }
        // ---- fetch ----------------------------------------------------------------------------
        const unsigned idle = __ballot_sync(MPG_FULL, !active);
        if (idle && more) {
            int got = 0;
            unsigned base = 0;
            const int want = __popc(idle);
            if (lane == 0) got = q_reserve(sh, PQ_RAY, want, base, r_end);
            got = __shfl_sync(MPG_FULL, got, 0);
            base = __shfl_sync(MPG_FULL, base, 0);
            if (got < want) more = false;   // the queue is exhausted: no more early exits from the traversal
            const int rank = __popc(idle & ((1u << lane) - 1u));
            if (!active && rank < got) {
                slot = q_take(pl, PQ_RAY, base + (unsigned)rank);
                const float *ry = pl.ray + slot;
                const int nv = pl.nv;
                const float3 o = f3(ry[0], ry[nv], ry[2 * nv]), d = f3(ry[3 * nv], ry[4 * nv], ry[5 * nv]);
                const float tmax = ry[6 * nv];
                const int hint = __float_as_int(ry[7 * nv]);
                any = hint == -2;
                spec_only = !any;
                rays++;
                best = tmax;
                bprim = -2; bsurf = -1;
                bb0 = bb1 = bb2 = 0.f;
                active = true;
                // analytic surfaces (as trace<W>)
                for (int i = 0; i < S.n_surf; i++) {
                    const DSurf &f = S.surf[i];
                    if (f.kind == 2 || (spec_only && f.mat == 2)) continue;
                    float t;
                    float3 p;
                    bool hit;
                    if (f.kind == 0) hit = sphere_hit(o, d, f.center, f.radius, eps, best, t, p);
                    else {
                        hit = quad_hit(o, d, f.origin, f.eu, f.ev, eps, best, t);
                        p = o + d * t;
                    }
                    if (hit) {
                        best = t; bprim = -1; bsurf = i; bp = p;
                        if (any) { active = false; break; }
                    }
                }
                node = SENT; leaf = NONE; sp = 1;
                if (active && S.n_tri > 0) {
                    ray_setup(r, o, d);
                    if (!any && hint >= 0) {   // bound the search by the hinted triangle (see trace<W>)
                        st.tris++;
                        const float4 p0 = __ldg(S.tpos + TSTRIDE * hint), p1 = __ldg(S.tpos + TSTRIDE * hint + 1),
                                     p2 = __ldg(S.tpos + TSTRIDE * hint + 2);
                        float t, c0, c1, c2;
                        if (!(spec_only && __float_as_int(p2.w) == 0) &&
                            tri_hit(r, xyz(p0), xyz(p1), xyz(p2), eps, best, t, c0, c1, c2)) {
                            best = t; bprim = hint; bsurf = __float_as_int(p1.w);
                            bb0 = c0; bb1 = c1; bb2 = c2;
                        }
                    }
                    oi = f3(o.x * r.idir.x, o.y * r.idir.y, o.z * r.idir.z);
                    stack[0] = SENT;
                    node = 0;
                } else {
                    active = false;
                }
                if (!active) fin = true;   // decided without the BVH
            }
        }
        if (!__any_sync(MPG_FULL, active)) {
            if (__any_sync(MPG_FULL, fin)) continue;   // flush the rays decided at fetch
            if (!more) break;
            continue;
        }
        // ---- traverse (while-while with postponed leaves) until `refill` lanes are idle -----
        while (true) {
            if (active) {
                while (node >= 0 && node != SENT) {
                    st.nodes++;
                    MPG_CHECK(node < S.n_nodes);
                    node = bvh_visit<W>(S.nodes, node, oi, r.idir, eps, best, stack, sp);
                    if (node < 0 && leaf == NONE) {
                        leaf = node;
                        node = stack[--sp];
                    }
                    if (!__any_sync(__activemask(), leaf == NONE)) break;
                }
                while (leaf != NONE) {
                    const int v = ~leaf;
                    const int start = v >> 3, cnt = (v & 7) + 1;
                    MPG_CHECK(start >= 0 && start + cnt <= S.n_tri);
                    for (int j = start; j < start + cnt; j++) {
                        st.tris++;
                        const float4 p0 = MPG_LDN(S.tpos + TSTRIDE * j), p1 = MPG_LDN(S.tpos + TSTRIDE * j + 1),
                                     p2 = MPG_LDN(S.tpos + TSTRIDE * j + 2);
                        if (spec_only && __float_as_int(p2.w) == 0) continue;
                        float t, c0, c1, c2;
                        if (tri_hit(r, xyz(p0), xyz(p1), xyz(p2), eps, best, t, c0, c1, c2)) {
                            best = t; bprim = j; bsurf = __float_as_int(p1.w);
                            bb0 = c0; bb1 = c1; bb2 = c2;
                            if (any) { node = SENT; break; }
                        }
                    }
                    leaf = NONE;
                    if (node < 0) {
                        leaf = node;
                        node = stack[--sp];
                    }
                    if (any && bsurf >= 0) { leaf = NONE; node = SENT; }
                }
                if (node == SENT && leaf == NONE) { active = false; fin = true; }
            }
            const unsigned act = __ballot_sync(MPG_FULL, active);
            if (act == 0u) break;
            if (more && 32 - __popc(act) >= refill) break;
        }
    }
}

// ---- rays of the three pass kinds (top of walk.cuh's trace_chain loop body) ----------------------
// reprojection ray ti of the chain in buffer cur, from `to` (x_D or the vertex just placed)
template <int KMAX, typename R>
__device__ __forceinline__ bool pool_build_reproj(Pool<KMAX, R> &pl, int slot, int cur, int ti, float beta, double3 to) {
    const double3 v = (pl.getx(cur, ti, slot) + tod(pl.getdq(ti, slot)) * (double)beta) - to;
    const double l2 = ddot(v, v);
    if (!(l2 > 0.0)) { pl.set_noray(slot, 3 | (ti << 4)); return false; }
    const double3 dd = v * rsqrt(l2);
    pl.set_ray(slot, f3d(to), nrmz(f3d(dd)), 3.0e38f, pl.getpr(cur, ti, slot));
    return true;
}
// visibility segment ti of the converged chain in buffer cur
template <int KMAX, typename R>
__device__ __forceinline__ void pool_build_vis(const WalkParams &P, Pool<KMAX, R> &pl, int slot, int cur, int k, int ti,
                                               float3 xD, uint32_t wi) {
    const float3 a = ti == 0 ? xD : f3d(pl.getx(cur, ti - 1, slot));
    const float3 b = ti == k ? xyz(__ldg(P.seed_xL + wi)) : f3d(pl.getx(cur, min(ti, KMAX - 1), slot));
    const float3 ab = b - a;
    const float l = len(ab);
    pl.set_ray(slot, a, ab * (1.0f / l), l - P.ray_eps, -2);
}
// deduction ray ti along dd (kept in the vertex's place of the chain being traced until its hit replaces it)
template <int KMAX, typename R>
__device__ __forceinline__ void pool_build_deduce(Pool<KMAX, R> &pl, int slot, int cur, int ti, double3 to, double3 dd) {
    pl.setx(cur ^ 1, ti, slot, dd);
    pl.set_ray(slot, f3d(to), nrmz(f3d(dd)), 3.0e38f, -1);
}

// ============================================================================
// hit phase: consume the hit of every slot in the hit queue (bottom of walk.cuh's trace_chain
// loop body), then either form the chain's next ray or end the pass (MPG_TRACE_TAIL): a
// complete chain goes to the Newton phase, a failed reprojection halves its step and
// re-enters the ray queue, everything else goes to the control phase
// ============================================================================
template <int KMAX, typename R, bool GL>
__device__ __forceinline__ void pool_hit(const DScene &S, const SeedCtx &g, const WalkParams &P, Pool<KMAX, R> &pl,
                                         PoolShared *sh, const int lane, int slot) {
    bool to_ray = false, to_hit = false, to_solve = false, to_ctl = false;
    if (slot >= 0) {
        const uint32_t ctw = pl.ct[slot], stw = pl.st[slot];
        const int k = (int)(ctw & 15u);
        const uint32_t bits = (ctw >> 12) & 255u;
        const bool learned = (ctw >> 20) & 1u;
        int cur = (int)((ctw >> 21) & 1u);
        int ti = CT_TI(ctw);
        uint32_t tau = (ctw >> 4) & 255u;   // deduction: the types resolved so far
        const int ph = ST_PH(stw);
        const int mode = ph == PH_DEDUCE ? TR_DEDUCE : (ph == PH_VIS ? TR_VIS : TR_REPROJ);
        int it = ST_IT(stw);
        float beta = pl.beta[slot];
        const float3 xD = pl.getxD(slot);
        const uint32_t wi = pl.w[slot];
        const int nv = pl.nv;
        const int hprim0 = __float_as_int(pl.ray[7 * nv + slot]);
        int tcode = 0;
        bool pass_end = false;
        if (hprim0 <= -16) {   // the ray could not be formed
            tcode = -(hprim0 + 16);
            pass_end = true;
        } else {
            const bool hit = hprim0 != -3;
            const int hsurf = __float_as_int(pl.ray[6 * nv + slot]);
            if (mode == TR_VIS) {
                if (hit) { tcode = 5; pass_end = true; }
                else if (++ti >= k + 1) pass_end = true;
                else { pool_build_vis(P, pl, slot, cur, k, ti, xD, wi); to_ray = true; }
            } else if (!hit) {
                tcode = 1 | (ti << 4);
                pass_end = true;
            } else if (mode == TR_REPROJ && hsurf != (int)((pl.sf[cur * nv + slot] >> (4 * ti)) & 15u)) {
                tcode = 2 | (ti << 4);
                pass_end = true;
            } else {
                if (mode == TR_DEDUCE) {
                    uint32_t bit = (bits >> ti) & 1u;
                    const int mat = S.surf[hsurf].mat;
                    if (!learned && mat == 0) bit = 0u;
                    if (bit && mat != 1) { tcode = 4 | (ti << 4); pass_end = true; }
                    else tau = (ti == 0 ? 0u : tau) | (bit << ti);
                }
                if (!pass_end) {
                    const double3 to = ti == 0 ? d3f(xD) : pl.getx(cur ^ 1, ti - 1, slot);
                    const double3 tdd = mode == TR_DEDUCE ? pl.getx(cur ^ 1, ti, slot) : make_double3(0.0, 0.0, 0.0);
                    int hprim = hprim0;
                    const float3 hp = f3(pl.ray[slot], pl.ray[nv + slot], pl.ray[2 * nv + slot]);
                    const double3 yi = refine_hit(S, hprim, hsurf, to,
                                                  mode == TR_DEDUCE
                                                      ? to + tdd
                                                      : pl.getx(cur, ti, slot) + tod(pl.getdq(ti, slot)) * (double)beta,
                                                  hp);
                    pl.setx(cur ^ 1, ti, slot, yi);
                    pl.setpr(cur ^ 1, ti, slot, hprim);
                    const uint32_t ysf = (ti == 0 ? 0u : pl.sf[(cur ^ 1) * nv + slot]) | ((uint32_t)(hsurf & 15) << (4 * ti));
                    pl.sf[(cur ^ 1) * nv + slot] = ysf;
                    if (++ti >= k) pass_end = true;
                    else if (mode == TR_REPROJ) {
                        if (pool_build_reproj(pl, slot, cur, ti, beta, yi)) to_ray = true;
                        else { tcode = 3 | (ti << 4); pass_end = true; }
                    } else {
                        double3 dd = tdd;
                        if (scatter_dir<GL>(S, dd, hprim, hsurf, yi, (tau >> (ti - 1)) & 1u, g.seed, P.walk_id_base + wi, ti - 1)) {
                            pool_build_deduce(pl, slot, cur, ti, yi, dd);
                            to_ray = true;
                        } else {
                            tcode = 4 | (ti << 4);
                            pass_end = true;
                        }
                    }
                }
            }
        }
        int phase = ph, end_status = ST_END(stw);
        bool occ = false;
        // ---- end of a pass (walk.cuh MPG_TRACE_TAIL) -------------------------
        while (pass_end) {
            pass_end = false;
            const bool ok = tcode == 0, ded = mode == TR_DEDUCE;
            if (mode == TR_VIS) {
                occ = !ok;
                phase = PH_END;
                to_ctl = true;
                break;
            }
            if (!ok && !ded && P.dbg && pl.trial[slot] == 0 && (int64_t)wi < P.n_dbg && 2 * it + 3 < P.dbg_stride)
                P.dbg[(int64_t)wi * P.dbg_stride + 2 * (it + 1)] = -(float)(tcode + 1);
            if (ok) {
                cur ^= 1;
                if (ded) { beta = P.beta0; it = 0; }   // tau = the resolved types
                else { beta = fminf(1.0f, 2.0f * beta); it++; }
                phase = PH_SOLVE;
                to_solve = true;
            } else if (ded) {
                end_status = ST_SEED_FAIL;
                phase = PH_END;
                to_ctl = true;
            } else {
                beta *= 0.5f;
                it++;
                if (it >= ((k >= 3 && P.max_iters_long > 0) ? P.max_iters_long : P.max_iters)) {
                    end_status = ST_MAXITER;
                    phase = PH_END;
                    to_ctl = true;
                } else {   // step halving: the same chain with the shorter step
                    ti = 0;
                    if (pool_build_reproj(pl, slot, cur, 0, beta, d3f(xD))) to_ray = true;
                    else { tcode = 3; pass_end = true; }
                }
            }
        }
        if (mode != TR_DEDUCE) tau = (ctw >> 4) & 255u;
        pl.ct[slot] = ct_pack(k, tau, bits, learned, cur, to_ray ? ti : 0);
        pl.st[slot] = st_pack(it, end_status, occ, ST_SEQ(stw), phase, ST_LID(stw));
        pl.beta[slot] = beta;
    }
    q_push(pl, sh, PQ_RAY, to_ray, slot, lane);
    q_push(pl, sh, PQ_SOLVE, to_solve, slot, lane);
    q_push(pl, sh, PQ_CTL, to_ctl, slot, lane);
    (void)to_hit;
}

// ============================================================================
// compute warps
// ============================================================================
template <int KMAX, typename R>
__device__ __forceinline__ void pool_load_chain(const Pool<KMAX, R> &pl, int slot, int cur, int k, double3 (&x)[KMAX],
                                                int (&prim)[KMAX], int (&surf)[KMAX]) {
    const uint32_t sfw = pl.sf[cur * pl.nv + slot];
#pragma unroll
    for (int i = 0; i < KMAX; i++) {
        if (i < k) {
            x[i] = pl.getx(cur, i, slot);
            prim[i] = pl.getpr(cur, i, slot);
        } else {
            x[i] = make_double3(0.0, 0.0, 0.0);
            prim[i] = -1;
        }
        surf[i] = (int)((sfw >> (4 * i)) & 15u);
    }
}

// Newton sweep on fresh chains (walk.cuh PH_SOLVE)
template <int KMAX, typename R, bool GL>
__device__ __forceinline__ void pool_solve(const DScene &S, const SeedCtx &g, const WalkParams &P, Pool<KMAX, R> &pl,
                                           PoolShared *sh, const int lane, int slot, uint32_t &c_vtx) {
    bool to_ray = false, to_ctl = false, to_hit = false;
    if (slot >= 0) {
        const uint32_t ctw = pl.ct[slot], stw = pl.st[slot];
        const int k = (int)(ctw & 15u), cur = (int)((ctw >> 21) & 1u);
        const uint32_t tau = (ctw >> 4) & 255u;
        const int it = ST_IT(stw), lid = ST_LID(stw);
        const uint32_t wi = pl.w[slot], trial = pl.trial[slot];
        const float3 xD = pl.getxD(slot);
        const float3 xL = xyz(__ldg(P.seed_xL + wi));
        double3 x[KMAX];
        int prim[KMAX], surf[KMAX];
        pool_load_chain(pl, slot, cur, k, x, prim, surf);
        c_vtx += k;
        float cm = 0.f;
        bool singular = false;
        R Di[KMAX][4], Ub[KMAX][4];
        V3<R> sg[KMAX], tg[KMAX], dq[KMAX];
        int phase = PH_REPROJ, end_status = 0;
        const int r = newton_system<KMAX, R, GL>(S, g.seed, P.walk_id_base + wi, k, tau, xD, xL, x, prim, surf, P.tol, Di,
                                                 Ub, sg, tg, dq, singular, cm);
        if (P.dbg && trial == 0 && (int64_t)wi < P.n_dbg && 2 * it + 1 < P.dbg_stride) {
            P.dbg[(int64_t)wi * P.dbg_stride + 2 * it] = cm;
            P.dbg[(int64_t)wi * P.dbg_stride + 2 * it + 1] = pl.beta[slot];
        }
        if (r == 1) {
            end_status = ST_CONVERGED;
            phase = PH_END;
            if (trial == 0) {
                const DLight &L = S.light[lid];
                float kap;
                R DL[4];
                if (!post_sweep<KMAX, R, GL>(S, g.seed, P.walk_id_base + wi, L, k, tau, xD, xL, x, prim, surf, true, kap,
                                             DL)) {
                    end_status = ST_BAD_SIDE;
                } else {
                    const float3 nD = xyz(__ldg(P.nD + wi / (uint32_t)P.spp));
                    const float Gc = singular ? 0.0f : ggt_from_blocks<KMAX, R>(k, xD, nD, x, Di, Ub, sg, tg, DL);
                    float Le = L.emit;
                    if (L.kind == 1 && !(dot(f3d(x[k - 1]) - xL, L.n) > 0.0f)) Le = 0.0f;
                    pl.Gc[slot] = Gc;
                    pl.Tc[slot] = kap * Gc * Le;
                    phase = PH_VIS;
                }
            }
        } else if (r == 2) {
            end_status = ST_DEGENERATE;
            phase = PH_END;
        } else {
            if (it >= ((k >= 3 && P.max_iters_long > 0) ? P.max_iters_long : P.max_iters)) {
                end_status = ST_MAXITER;
                phase = PH_END;
            } else {
#pragma unroll
                for (int i = 0; i < KMAX; i++)
                    if (i < k) pl.setdq(i, slot, dq[i]);
            }
        }
        pl.st[slot] = st_pack(it, end_status, false, ST_SEQ(stw), phase, lid);
        to_ctl = phase == PH_END;
        // the first ray of the next pass: reprojection ray 0, or visibility segment 0
        if (phase == PH_VIS) {
            pool_build_vis(P, pl, slot, cur, k, 0, xD, wi);
            to_ray = true;
        } else if (phase == PH_REPROJ) {
            if (pool_build_reproj(pl, slot, cur, 0, pl.beta[slot], d3f(xD))) to_ray = true;
            else to_hit = true;   // no ray: the hit phase ends the pass (step halving)
        }
    }
    q_push(pl, sh, PQ_RAY, to_ray, slot, lane);
    q_push(pl, sh, PQ_HIT, to_hit, slot, lane);
    q_push(pl, sh, PQ_CTL, to_ctl, slot, lane);
}

// End-of-attempt bookkeeping, trials, fetch, seeds (walk.cuh PH_END / PH_FETCH / PH_WAIT / PH_SEED)
// for the slots of one control or wait batch.  Returns true if any lane made progress.
template <int KMAX, typename R, bool GL>
__device__ __forceinline__ bool pool_control(const DScene &S, const SeedCtx &g, const WalkParams &P, Pool<KMAX, R> &pl,
                                             PoolShared *sh, const int lane, int slot, uint32_t &c_newton,
                                             uint32_t &c_attempts) {
    unsigned *s_stats = sh->stats;
    // slot state in registers for the batch
    int phase = PH_IDLE;
    int64_t w = -1;
    uint32_t trial = 0, psurf = 0, ptau = 0, tau = g.tau, ticket = 0xffffffffu;
    int k = g.k, pk = g.k, cur = 0, it = 0, end_status = 0, lid = 0, item_e = -1;
    bool occluded = false, seq_only = false;
    float Tprim = 0.f, pdfL = 1.f;
    float3 xD = f3(0.f, 0.f, 0.f), xL = f3(0.f, 0.f, 0.f);
    uint32_t my_resolved = 0;
    bool progress = false;
    if (slot >= 0) {
        const uint32_t ctw = pl.ct[slot], stw = pl.st[slot];
        phase = ST_PH(stw);
        it = ST_IT(stw);
        end_status = ST_END(stw);
        occluded = ST_OCC(stw);
        seq_only = ST_SEQ(stw);
        lid = ST_LID(stw);
        k = (int)(ctw & 15u);
        tau = (ctw >> 4) & 255u;
        cur = (int)((ctw >> 21) & 1u);
        trial = pl.trial[slot];
        item_e = pl.item_e[slot];
        ticket = pl.ticket[slot];
        if (phase == PH_END) {
            w = (int64_t)pl.w[slot];
            const uint32_t pct = pl.pct[slot];
            pk = (int)(pct & 15u);
            ptau = pct >> 4;
            psurf = pl.psurf[slot];
            Tprim = pl.Tprim[slot];
            xD = pl.getxD(slot);
            const float4 l4 = __ldg(P.seed_xL + w);
            xL = xyz(l4);
            pdfL = l4.w;
        }
    }
    float3 tgt = f3(0.f, 0.f, 0.f);
    uint32_t bits = g.tau;
    bool learned = true;
    bool to_ray = false, to_wait = false, to_hit = false;
    while (true) {
        // ---- end of an attempt -------------------------------------------------
        if (phase == PH_END) {
            progress = true;
            c_newton += (uint32_t)it;
            int st = end_status;
            if (trial == 0) {
                float G = 0.f, T = 0.f;
                if (st == ST_CONVERGED) {
                    if (occluded) st = ST_OCCLUDED;
                    else { G = pl.Gc[slot]; T = pl.Tc[slot]; }
                }
                uint32_t sfw = 0;
                if (st != ST_SEED_FAIL && st != ST_INACTIVE) {
                    sfw = pl.sf[cur * pl.nv + slot];
#pragma unroll
                    for (int i = 0; i < KMAX; i++) {
                        if (i >= k) break;
                        const int pi = pl.getpr(cur, i, slot);
                        const double3 xi = pl.getx(cur, i, slot);
                        int pid = pi >= 0 ? __float_as_int(__ldg(S.tpos + TSTRIDE * pi).w) : -1;
                        MPG_CHECK(w >= 0 && w < P.n && i < KMAX);
                        P.chain[(int64_t)i * P.n + w] = make_float4((float)xi.x, (float)xi.y, (float)xi.z, __int_as_float(pid));
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
                        psurf |= ((sfw >> (4 * i)) & 15u) << (4 * i);
                    }
                    if (P.psurf_out) P.psurf_out[w] = psurf;
                    const bool dr = *(volatile unsigned *)&sh->drained != 0u;
                    if (queue_drained(P, dr) && P.items && hard_publish(P, w, psurf, pk, ptau, 0u, seq_only))
                        phase = PH_FETCH;
                    else {
                        trial = 1;
                        phase = PH_SEED;
                    }
                } else {
                    P.trials[w] = 0;
                    P.w[w] = 0.0f;
                    my_resolved++;
                    phase = PH_FETCH;
                }
            } else {
                bool same = false;
                if (st == ST_CONVERGED && k == pk && tau == ptau) {
                    double3 x[KMAX];
                    int prim[KMAX], surf[KMAX];
                    pool_load_chain(pl, slot, cur, k, x, prim, surf);
                    float kdummy;
                    R DLdummy[4];
                    if (post_sweep<KMAX, R, GL>(S, g.seed, P.walk_id_base + w, S.light[lid], k, tau, xD, xL, x, prim, surf,
                                                false, kdummy, DLdummy)) {
                        same = true;
#pragma unroll
                        for (int i = 0; i < KMAX; i++) {
                            if (i >= k) break;
                            float4 c = __ldcg(P.chain + (int64_t)i * P.n + w);
                            float3 dd = f3d(x[i]) - xyz(c);
                            if ((int)((psurf >> (4 * i)) & 15u) != (surf[i] & 15) || !(len(dd) < P.same_eps)) same = false;
                        }
                    }
                }
                const bool dr = *(volatile unsigned *)&sh->drained != 0u;
                if (item_e >= 0) {
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
                            my_resolved++;
                        } else if (issued >= P.k_max) {
                            trial_finalize(P, w, P.k_max, true, s_stats);
                            my_resolved++;
                        } else {
                            const unsigned backlog = *(volatile unsigned *)&P.th->item_tail -
                                                     *(volatile unsigned *)&P.th->item_head;
                            const uint32_t gr = (int)backlog < (int)P.idle_backlog && queue_drained(P, dr) ? P.item_grow_idle
                                                                                                          : P.item_grow;
                            const uint32_t B = min(__ldcg(P.e_batch + e) << gr, P.k_max - issued);
                            P.e_batch[e] = B;
                            P.e_pending[e] = B;
                            P.e_issued[e] = issued + B;
                            __threadfence();
                            if (!items_push(P, e, issued + 1, B)) {
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
                    my_resolved++;
                    phase = PH_FETCH;
                } else {
                    if ((trial >= P.local_trials || queue_drained(P, dr)) && !seq_only && P.items &&
                        hard_publish(P, w, psurf, pk, ptau, trial, seq_only))
                        phase = PH_FETCH;
                    else {
                        trial++;
                        phase = PH_SEED;
                    }
                }
            }
        }
        // ---- fetch a primary walk (warp-aggregated) ------------------------------
        const unsigned need = __ballot_sync(MPG_FULL, phase == PH_FETCH);
        if (need) {
            progress = true;
            const int leader = __ffs(need) - 1;
            unsigned long long base = 0;
            if (lane == leader) {
                base = atomicAdd(&P.th->queue, (unsigned long long)__popc(need));
                if (base + __popc(need) >= (unsigned long long)P.n) *(volatile unsigned *)&sh->drained = 1u;
            }
            base = __shfl_sync(MPG_FULL, base, leader);
            if (phase == PH_FETCH) {
                const int64_t idx = (int64_t)base + __popc(need & ((1u << lane) - 1u));
                item_e = -1;
                seq_only = false;
                if (idx < P.n) {
                    w = P.perm ? (int64_t)__ldg(P.perm + idx) : idx;
                    trial = 0;
                    xD = xyz(__ldg(P.xD + w / P.spp));
                    const float4 l4 = __ldg(P.seed_xL + w);
                    xL = xyz(l4);
                    pdfL = l4.w;
                    lid = 0;
                    if (S.n_light > 1) lid = (int)uidx(rng_draw(g.seed, P.walk_id_base + w, 0u, 0u).z, (uint32_t)S.n_light);
                    phase = PH_SEED;
                    if (P.trials_only) {
                        const float T0 = P.T[w];
                        if (P.status[w] == ST_CONVERGED && T0 > 0.0f && P.trials_on) {
                            const uint32_t c2 = P.out_ctype ? (uint32_t)P.out_ctype[w] : ((uint32_t)g.k | (g.tau << 4));
                            pk = (int)(c2 & 15u);
                            ptau = c2 >> 4;
                            psurf = P.psurf_out[w];
                            Tprim = T0;
                            trial = 1;
                        } else {
                            P.trials[w] = 0;
                            P.w[w] = 0.0f;
                            my_resolved++;
                            phase = PH_FETCH;
                        }
                    }
                } else {
                    phase = PH_WAIT;
                    ticket = 0xffffffffu;
                }
            }
        }
        // ---- trial items by ticket ------------------------------------------------
        {
            const unsigned needt = __ballot_sync(MPG_FULL, phase == PH_WAIT && ticket == 0xffffffffu);
            if (needt) {
                const int leader = __ffs(needt) - 1;
                unsigned base = 0;
                if (lane == leader) base = atomicAdd(&P.th->item_head, (unsigned)__popc(needt));
                base = __shfl_sync(MPG_FULL, base, leader);
                if (phase == PH_WAIT && ticket == 0xffffffffu) ticket = base + (unsigned)__popc(needt & ((1u << lane) - 1u));
            }
        }
        if (phase == PH_WAIT) {
            const unsigned long long wd =
                ticket < P.item_cap ? *(volatile unsigned long long *)(P.items + ticket) : ITEM_EMPTY;
            if (wd != ITEM_EMPTY) {
                progress = true;
                ticket = 0xffffffffu;
                item_e = (int)(wd >> 32);
                trial = (uint32_t)wd;
                MPG_CHECK(item_e >= 0 && (uint32_t)item_e < P.hard_cap);
                w = __ldcg(P.e_walk + item_e);
                MPG_CHECK(w >= 0 && w < P.n);
                psurf = __ldcg(P.e_psurf + item_e);
                const uint32_t pct = __ldcg(P.e_pct + item_e);
                pk = (int)(pct & 15u);
                ptau = pct >> 4;
                xD = xyz(__ldg(P.xD + w / P.spp));
                const float4 l4 = __ldg(P.seed_xL + w);
                xL = xyz(l4);
                pdfL = l4.w;
                lid = 0;
                if (S.n_light > 1) lid = (int)uidx(rng_draw(g.seed, P.walk_id_base + w, 0u, 0u).z, (uint32_t)S.n_light);
                if (*(volatile uint32_t *)(P.e_best + item_e) < trial) { end_status = ST_SEED_FAIL; it = 0; phase = PH_END; }
                else phase = PH_SEED;
            } else {
                if (*(volatile unsigned int *)&P.th->resolved >= (unsigned int)P.n) *(volatile unsigned *)&sh->done = 1u;
                to_wait = true;   // park the slot again
            }
        }
        // ---- seed -------------------------------------------------------------------
        if (phase == PH_SEED) {
            c_attempts++;
            bool ok;
            bool inactive = false;
            if (trial == 0) {
                const int sb = __ldg(P.seed_bin + w);
                ok = sb >= -1;
                inactive = sb == -3;
                tgt = xyz(__ldg(P.seed_tgt + w));
                k = g.k;
                bits = g.tau;
                learned = true;
                if (P.seed_ctype) {
                    const uint32_t c2 = __ldg(P.seed_ctype + w);
                    k = (int)(c2 & 15u);
                    bits = (c2 >> 4) & 255u;
                    learned = (c2 >> 12) & 1u;
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
            if (ok) {
                phase = PH_DEDUCE;
                to_ray = true;
            } else {
                end_status = inactive ? ST_INACTIVE : ST_SEED_FAIL;
                phase = PH_END;
            }
        }
        if (!__any_sync(MPG_FULL, phase == PH_END || phase == PH_FETCH || phase == PH_SEED)) break;
    }
    // ---- store the slots and hand them on --------------------------------------------
    if (slot >= 0) {
        if (to_ray) {
            pl.w[slot] = (uint32_t)w;
            pl.trial[slot] = trial;
            pl.ct[slot] = ct_pack(k, g.tau, bits, learned, 0);
            pl.pct[slot] = (uint32_t)pk | (ptau << 4);
            pl.psurf[slot] = psurf;
            pl.Tprim[slot] = Tprim;
            pl.item_e[slot] = item_e;
            pl.beta[slot] = P.beta0;
            pl.setxD(slot, xD);
            pl.sf[slot] = 0u;
            pl.st[slot] = st_pack(0, 0, false, seq_only, PH_DEDUCE, lid);
            // deduction ray 0: x_D towards the seed target (Eq. 6)
            const double3 v = d3f(tgt) - d3f(xD);
            const double l2 = ddot(v, v);
            if (!(l2 > 0.0)) { pl.set_noray(slot, 3); to_hit = true; }
            else pool_build_deduce(pl, slot, 0, 0, d3f(xD), v * rsqrt(l2));
        } else {
            pl.ticket[slot] = ticket;
            pl.st[slot] = st_pack(0, 0, false, false, PH_WAIT, 0);
        }
    }
    // walks made final by this batch: one atomic per warp, after their outputs
    const unsigned tot = __reduce_add_sync(MPG_FULL, my_resolved);
    if (tot) {
        __threadfence();
        if (lane == 0) atomicAdd(&P.th->resolved, tot);
    }
    q_push(pl, sh, PQ_RAY, to_ray && !to_hit, slot, lane);
    q_push(pl, sh, PQ_HIT, to_ray && to_hit, slot, lane);
    q_push(pl, sh, PQ_WAIT, slot >= 0 && !to_ray, slot, lane);
    (void)pdfL;
    (void)to_wait;
    return progress;
}

// One block per SM, NW universal warps.  The block cycles through three phases separated by
// barriers, so that at any time all its warps execute the same (instruction-cache-sized) code:
//   T  trace one pass of every slot in the ray queue,
//   S  Newton sweep of every slot with a fresh chain,
//   C  end-of-attempt bookkeeping / trials / fetch / seeds of every slot in the control queue,
//      and one poll of the trial-item ring for the waiting slots.
#ifndef MPG_POOL_BPS
#define MPG_POOL_BPS 1   // blocks per SM
#endif
template <int KMAX, typename R, int W, bool GL, int NW>
__global__ void __launch_bounds__(NW * 32, MPG_POOL_BPS)
    k_walk_pool(const DScene S, const SeedCtx g, const WalkParams P, const int nv, const int nvq, const int s_min,
                const int c_min, const int refill, unsigned char *gstate) {
    extern __shared__ __align__(16) unsigned char pool_smem[];
    __shared__ PoolShared sh;
    Pool<KMAX, R> pl;
    // slot state in shared memory, or (gstate) in this block's region of a global buffer (L2-resident)
    if (gstate) pl.carve(gstate + (size_t)blockIdx.x * (((size_t)Pool<KMAX, R>::slot_bytes() * nv + 255) & ~(size_t)255), pool_smem, nv, nvq);
    else pl.carve(pool_smem, nullptr, nv, nvq);
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < PQ_N) { sh.head[threadIdx.x] = 0u; sh.tail[threadIdx.x] = 0u; }
    if (threadIdx.x == 0) { sh.done = 0u; sh.drained = 0u; }
    for (int i = threadIdx.x; i < SS_N; i += blockDim.x) sh.stats[i] = 0u;
    for (int i = threadIdx.x; i < PQ_N * nvq; i += blockDim.x) pl.ring[i] = 0;
    __syncthreads();
    // every slot starts in the control queue, asking for a primary walk
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
        pl.st[i] = st_pack(0, 0, false, false, PH_FETCH, 0);
        pl.ct[i] = ct_pack(g.k, g.tau, g.tau, true, 0);
        pl.trial[i] = 0u;
        pl.item_e[i] = -1;
        pl.ticket[i] = 0xffffffffu;
        pl.ring[(size_t)PQ_CTL * nvq + i] = (unsigned short)(i + 1);
    }
    if (threadIdx.x == 0) sh.tail[PQ_CTL] = (unsigned)nv;
    __syncthreads();

    LaneStats ls = {0u, 0u, 0u};
    unsigned long long rays = 0;
    uint32_t c_newton = 0, c_attempts = 0, c_vtx = 0;
    unsigned backoff = 256u;
    if (threadIdx.x == 0) { sh.sel = PS_CTL; sh.progress = 1u; }
    for (int q = threadIdx.x; q < PQ_N; q += blockDim.x) sh.end[q] = 0u;
    PROF_DECL
    while (true) {
        // ---- scheduler: thread 0 picks the next phase from the queue lengths ---------------
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < PQ_N; q++)   // undo reservation overshoots of the last phase
                if ((int)(sh.head[q] - sh.end[q]) > 0) sh.head[q] = sh.end[q];
            const int nR = (int)(sh.tail[PQ_RAY] - sh.head[PQ_RAY]), nH = (int)(sh.tail[PQ_HIT] - sh.head[PQ_HIT]),
                      nS = (int)(sh.tail[PQ_SOLVE] - sh.head[PQ_SOLVE]), nC = (int)(sh.tail[PQ_CTL] - sh.head[PQ_CTL]);
            unsigned sel;
            if (sh.done) sel = PS_EXIT;
            else if (nH > 0) sel = PS_HIT;
            else if (nS >= s_min) sel = PS_SOLVE;
            else if (nC >= c_min) sel = PS_CTL;
            else if (nR > 0) sel = PS_TRACE;
            else if (nS > 0) sel = PS_SOLVE;
            else if (nC > 0) sel = PS_CTL;
            else sel = sh.progress ? PS_CTL : PS_SLEEP;   // only waiting slots: poll (with back-off)
            for (int q = 0; q < PQ_N; q++) sh.end[q] = sh.head[q];
            if (sel == PS_TRACE) sh.end[PQ_RAY] = sh.tail[PQ_RAY];
            if (sel == PS_HIT) sh.end[PQ_HIT] = sh.tail[PQ_HIT];
            if (sel == PS_SOLVE) sh.end[PQ_SOLVE] = sh.tail[PQ_SOLVE];
            if (sel == PS_CTL || sel == PS_SLEEP) { sh.end[PQ_CTL] = sh.tail[PQ_CTL]; sh.end[PQ_WAIT] = sh.tail[PQ_WAIT]; }
            sh.progress = 0u;
            sh.sel = sel;
        }
        __syncthreads();
        const unsigned sel = sh.sel;
        PROF_LAP(11)
        if (sel == PS_EXIT) break;
        if (sel == PS_TRACE) {
            // ---- R: the ray of every slot in the ray queue ----------------------------------
            pool_ray_phase<KMAX, R, W>(S, P, pl, &sh, lane, sh.end[PQ_RAY], refill, rays, ls);
            PROF_LAP(2)
            PROF_ADD(0, 1);
        } else if (sel == PS_HIT) {
            // ---- H: consume the hits, form the next rays or end the passes ---------------
            const unsigned h_end = sh.end[PQ_HIT];
            while (true) {
                int got = 0;
                unsigned base = 0;
                if (lane == 0) got = q_reserve(&sh, PQ_HIT, 32, base, h_end);
                got = __shfl_sync(MPG_FULL, got, 0);
                base = __shfl_sync(MPG_FULL, base, 0);
                if (!got) break;
                const int slot = lane < got ? q_take(pl, PQ_HIT, base + (unsigned)lane) : -1;
                pool_hit<KMAX, R, GL>(S, g, P, pl, &sh, lane, slot);
            }
            PROF_LAP(3)
            PROF_ADD(12, 1);
        } else if (sel == PS_SOLVE) {
            // ---- S: Newton sweep of the fresh chains --------------------------------------
            const unsigned s_end = sh.end[PQ_SOLVE];
            while (true) {
                int got = 0;
                unsigned base = 0;
                if (lane == 0) got = q_reserve(&sh, PQ_SOLVE, 32, base, s_end);
                got = __shfl_sync(MPG_FULL, got, 0);
                base = __shfl_sync(MPG_FULL, base, 0);
                if (!got) break;
                const int slot = lane < got ? q_take(pl, PQ_SOLVE, base + (unsigned)lane) : -1;
                pool_solve<KMAX, R, GL>(S, g, P, pl, &sh, lane, slot, c_vtx);
                PROF_ADD(5, 1);
                PROF_ADD(6, got);
            }
            PROF_LAP(7)
            PROF_ADD(1, 1);
        } else {
            // ---- C: control queue, then one poll of the waiting slots ---------------------
            if (sel == PS_SLEEP) {
                __nanosleep(backoff);
                backoff = min(2u * backoff, P.backoff_max);
            } else {
                backoff = 256u;
            }
            bool progress = false;
            for (int q = PQ_CTL; q <= PQ_WAIT; q++) {
                const unsigned q_end = sh.end[q];   // slots re-parked in this phase wait for the next
                while (true) {
                    int got = 0;
                    unsigned base = 0;
                    if (lane == 0) got = q_reserve(&sh, q, 32, base, q_end);
                    got = __shfl_sync(MPG_FULL, got, 0);
                    base = __shfl_sync(MPG_FULL, base, 0);
                    if (!got) break;
                    const int slot = lane < got ? q_take(pl, q, base + (unsigned)lane) : -1;
                    progress |= pool_control<KMAX, R, GL>(S, g, P, pl, &sh, lane, slot, c_newton, c_attempts);
                    PROF_ADD(8, 1);
                    PROF_ADD(9, got);
                }
            }
            if (__any_sync(MPG_FULL, progress) && lane == 0) *(volatile unsigned *)&sh.progress = 1u;
            PROF_LAP(10)
            PROF_ADD(4, 1);
        }
    }
    PROF_FLUSH
    // ---- stats reduction ----------------------------------------------------
    unsigned long long v[6] = {c_newton, c_attempts, rays, ls.nodes, ls.tris, c_vtx};
#pragma unroll
    for (int j = 0; j < 6; j++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(MPG_FULL, v[j], o);
    }
    if (lane == 0 && P.stats) {
        if (v[0]) atomicAdd(P.stats + SS_NEWTON, v[0]);
        if (v[1]) atomicAdd(P.stats + SS_ATTEMPTS, v[1]);
        if (v[2]) atomicAdd(P.stats + SS_RAYS, v[2]);
        if (v[3]) atomicAdd(P.stats + SS_NODES, v[3]);
        if (v[4]) atomicAdd(P.stats + SS_TRIS, v[4]);
        if (v[5]) atomicAdd(P.stats + SS_VTX, v[5]);
    }
    __syncthreads();
    if (P.stats)
        for (int i = threadIdx.x; i < SS_N; i += blockDim.x)
            if (sh.stats[i]) atomicAdd(P.stats + i, (unsigned long long)sh.stats[i]);
}
