// stree.cuh -- the paper's own guide on the GPU: an STree over the
// 6D configuration (x_D, x_L) with per-leaf length / type tables and vMF mixtures
// of the solved directions (§5.5-5.6; Eqs. 9-13; readings
// R28-R31 in DESIGN.md).  Included by mpg.cu after the histogram guide.
//
// Build (mpg_guide_rebuild), level-synchronous and deterministic:
//   k_stree_valid      flags + exact fp32 bbox of the sample keys (warp min/max, atomics)
//   DeviceSelect       ids of the samples, record order
//   per level          one pinned upload of the level's node table; keys (node index << 32 |
//                      ordered coordinate) and one stable cub radix sort of (key, id) = every
//                      node's list stably sorted by the split axis; k_stree_split (one thread
//                      per node: plane, overlap windows by binary search); one D2H + sync;
//                      the host lays out the child windows (prefix sums over a few thousand
//                      nodes) and k_copy_segments (element-parallel) writes the next level
//   lobes              radix sort by (leaf, type, position) = stable partition by type;
//                      k_grp_off, k_lobe_kappa (nearest direction in the group),
//                      k_group_tables (E_tau in fp64, integer lobe weights), then the
//                      per-leaf length / type tables of the histogram guide (k_dir_cell_tables)
// Children are contiguous windows of the parent's sorted list, so the build is a
// sequence of sorts and copies; no atomics decide anything.
#pragma once
#include <chrono>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

template <class T> struct DBuf {
    T *p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t n) { // contents not kept
        if (n <= cap && p) return cudaSuccess;
        cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t c = std::max<size_t>(n, 1) * 5 / 4 + 16;
        cudaError_t e = cudaMalloc(&p, c * sizeof(T));
        if (e == cudaSuccess) cap = c;
        return e;
    }
    cudaError_t reserve_keep(size_t n, size_t used, cudaStream_t s) {
        if (n <= cap && p) return cudaSuccess;
        T *q = nullptr;
        size_t c = std::max<size_t>(n, 1) * 3 / 2 + 16;
        cudaError_t e = cudaMalloc(&q, c * sizeof(T));
        if (e != cudaSuccess) return e;
        if (used) e = cudaMemcpyAsync(q, p, used * sizeof(T), cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(p);
        p = q;
        cap = c;
        return e;
    }
    void release() {
        cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

template <class T> struct PinBuf { // pinned host staging (reused; rewritten only after a stream sync)
    T *p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t c = std::max<size_t>(n, 1) * 3 / 2 + 64;
        cudaError_t e = cudaHostAlloc((void **)&p, c * sizeof(T), cudaHostAllocDefault);
        if (e == cudaSuccess) cap = c;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

struct StreeState {
    mpg_stree_desc d;
    const float4 *sep_wv = nullptr, *sep_n = nullptr; // glossy separator (Eq. 14): per receiver
    float sep_alpha = 0.f;
    DBuf<mpg_guide_sample> rec;
    int64_t n_rec = 0;
    // current tree
    int root_ref = ~0, n_nodes = 0, n_leaves = 0, thr = 1;
    int64_t n_valid = 0, n_lobes = 0;
    DBuf<int4> nodes;
    DBuf<int64_t> leaf_begin, leaf_count;
    DBuf<int> leaf_ids, grp_off, lobe_sample;
    DBuf<unsigned long long> lobe_prefix;
    DBuf<float4> lobe_mu;
    DBuf<uint64_t> n_prefix, type_prefix;
    DBuf<int> leaf_own;                  // [leaves] own (non-copy) samples (selective activation, R36)
    DBuf<double> E;
    // scratch
    DBuf<unsigned char> flags;
    DBuf<int> ids_a, ids_b, ids_c, nv;
    DBuf<unsigned long long> keys_a, keys_b;
    DBuf<unsigned char> temp;
    DBuf<unsigned int> bbox;
    DBuf<int4> split_out;
    DBuf<int4> dstage_a, dstage_b;    // per-level device staging (level data, child segments)
    PinBuf<int4> hstage_a, hstage_b;  // pinned host staging of the same
    PinBuf<int4> hsplit;              // split results (m, eL, eR, s0 | s1, c bits)
};

static void stree_state_free(StreeState *t) {
    if (!t) return;
    t->rec.release(); t->nodes.release(); t->leaf_begin.release(); t->leaf_count.release();
    t->leaf_ids.release(); t->grp_off.release(); t->lobe_sample.release(); t->lobe_prefix.release();
    t->lobe_mu.release(); t->n_prefix.release(); t->type_prefix.release(); t->leaf_own.release(); t->E.release();
    t->flags.release(); t->ids_a.release(); t->ids_b.release(); t->ids_c.release();
    t->nv.release(); t->keys_a.release(); t->keys_b.release(); t->temp.release(); t->bbox.release();
    t->split_out.release();
    t->dstage_a.release(); t->dstage_b.release(); t->hstage_a.release(); t->hstage_b.release(); t->hsplit.release();
    delete t;
}

__device__ __forceinline__ bool gs_valid(const mpg_guide_sample &r) { return r.w > 0.0f && r.type >= 0 && r.type < 126; }
__device__ __forceinline__ float gs_key(const mpg_guide_sample &r, int a) {
    return canon0(a < 3 ? r.xD[a] : r.xL[a - 3]);
}
// order-preserving float <-> u32 (keys never hold -0, R28)
__device__ __forceinline__ unsigned f2o(float x) {
    unsigned u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float o2f(unsigned u) { return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u); }

// sample flags and the exact fp32 bbox of the keys (min/max are order-independent)
__global__ void k_stree_valid(const mpg_guide_sample *rec, int64_t n, unsigned char *flags, unsigned *bbox) {
    unsigned mn[6], mx[6];
#pragma unroll
    for (int a = 0; a < 6; a++) { mn[a] = 0xffffffffu; mx[a] = 0u; }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        mpg_guide_sample r = rec[i];
        bool v = gs_valid(r);
        flags[i] = v ? 1 : 0;
        if (v) {
#pragma unroll
            for (int a = 0; a < 6; a++) {
                unsigned o = f2o(gs_key(r, a));
                mn[a] = min(mn[a], o);
                mx[a] = max(mx[a], o);
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 6; a++) {
        unsigned m0 = __reduce_min_sync(MPG_FULL, mn[a]), m1 = __reduce_max_sync(MPG_FULL, mx[a]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(bbox + a, m0);
            atomicMax(bbox + 6 + a, m1);
        }
    }
}

// element-parallel: key = (node index in the level) << 32 | ordered coordinate; a stable
// radix sort of (key, id) then orders every node's list by the coordinate, equal
// coordinates keeping the list's order (R29).  nodes: (begin, count), contiguous.
__global__ void k_level_keys(const mpg_guide_sample *rec, const int *ids, int64_t n, const int2 *nodes, int nl,
                             int axis, unsigned long long *keys) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nl - 1; // last node with begin <= j
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (nodes[mid].x <= (int)j) lo = mid;
            else hi = mid - 1;
        }
        int id = ids[j];
        keys[j] = ((unsigned long long)lo << 32) | f2o(gs_key(rec[id], axis));
    }
}

// one thread per splitting node (R28, R29): plane c, copies eL/eR, discard bounds s0/s1
__global__ void k_stree_split(const unsigned long long *keys, const int2 *sbe, const float2 *lohi, int n_nodes,
                              float eps, int4 *out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_nodes) return;
    const unsigned long long *K = keys + sbe[t].x;
    int k = sbe[t].y - sbe[t].x;
    // keys: low word = ordered coordinate
    float lo = lohi[t].x, hi = lohi[t].y;
    float c = FM(FA(lo, hi), 0.5f);
    float delta = FM(FS(hi, lo), 0.25f);
    auto x = [&](int j) { return o2f((unsigned)K[j]); };
    // first index in [a, b) where pred holds, pred monotone false..true
    auto first = [&](int a, int b, auto pred) {
        while (a < b) {
            int mid = (a + b) >> 1;
            if (pred(mid)) b = mid;
            else a = mid + 1;
        }
        return a;
    };
    int m = first(0, k, [&](int j) { return !(x(j) < c); });
    long long E = (long long)floor((double)eps * (double)k);
    int cR = first(m, k, [&](int j) { return FS(x(j), c) > delta; }) - m;
    int cL = m - first(0, m, [&](int j) { return FS(c, x(j)) <= delta; });
    int eR = (int)min((long long)cR, E), eL = (int)min((long long)cL, E);
    int s0 = first(0, m, [&](int j) { return FS(lo, x(j)) <= delta; });
    int s1 = first(m, k, [&](int j) { return FS(x(j), hi) > delta; });
    out[2 * t] = make_int4(m, eL, eR, s0);
    out[2 * t + 1] = make_int4(s1, __float_as_int(c), 0, 0);
}

// element-parallel copy of segments (src, dst, len) whose dst ranges are contiguous and
// increasing from segs[0].y: total elements n
__global__ void k_copy_segments(const int *src, int *dst, const int4 *segs, int nseg, int64_t n) {
    const int d0 = segs[0].y;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        int d = d0 + (int)e;
        int lo = 0, hi = nseg - 1; // last segment with dst <= d
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (segs[mid].y <= d) lo = mid;
            else hi = mid - 1;
        }
        int4 g = segs[lo];
        dst[d] = src[g.x + (d - g.y)];
    }
}

__global__ void k_lobe_keys(const mpg_guide_sample *rec, const int *leaf_ids, const int64_t *lb, const int64_t *lc,
                            unsigned long long *keys) {
    int l = blockIdx.x;
    int64_t b = lb[l], n = lc[l];
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        int64_t pos = b + j;
        keys[pos] = ((unsigned long long)l << 40) | ((unsigned long long)rec[leaf_ids[pos]].type << 32) |
                    (unsigned long long)(unsigned)pos;
    }
}

__global__ void k_lobe_sample(const unsigned long long *keys, const int *leaf_ids, int64_t n, int *lobe_sample) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        lobe_sample[j] = leaf_ids[(unsigned)keys[j]];
}

// grp_off[leaf][t] = first lobe with (leaf, type) >= (leaf, t), t = 0..126
__global__ void k_grp_off(const unsigned long long *keys, int64_t n, int n_leaves, int *grp_off) {
    int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n_leaves * 127) return;
    unsigned long long q = ((unsigned long long)(id / 127) << 40) | ((unsigned long long)(id % 127) << 32);
    int64_t a = 0, b = n;
    while (a < b) {
        int64_t mid = (a + b) >> 1;
        if (keys[mid] >= q) b = mid;
        else a = mid + 1;
    }
    grp_off[id] = (int)a;
}

// vMF lobes (R30): mu = w_D*, kappa = 1 / (nearest chord distance)^2 in the (leaf, type) group
__global__ void k_lobe_kappa(const mpg_guide_sample *rec, const unsigned long long *keys, const int *lobe_sample,
                             const int *grp_off, int64_t n, float kmin, float kmax, float4 *lobe_mu) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long key = keys[j];
        int g = (int)(key >> 40) * 127 + (int)((key >> 32) & 0xffu);
        int glo = grp_off[g], ghi = grp_off[g + 1];
        const mpg_guide_sample &ri = rec[lobe_sample[j]];
        float ox = ri.omega[0], oy = ri.omega[1], oz = ri.omega[2];
        float d2min = __int_as_float(0x7f800000);
        for (int q = glo; q < ghi; q++) {
            if (q == (int)j) continue;
            const mpg_guide_sample &rj = rec[lobe_sample[q]];
            float dx = FS(ox, rj.omega[0]), dy = FS(oy, rj.omega[1]), dz = FS(oz, rj.omega[2]);
            float d2 = FA(FA(FM(dx, dx), FM(dy, dy)), FM(dz, dz));
            d2min = fminf(d2min, d2);
        }
        // Eq. 12: kappa = sigma'^-2; a lone lobe takes 1, sigma' = 0 takes kmax (R30)
        float kap = ghi - glo == 1 ? 1.0f : (d2min > 0.0f ? FD(1.0f, d2min) : kmax);
        kap = fminf(fmaxf(kap, kmin), kmax);
        lobe_mu[j] = make_float4(ox, oy, oz, kap);
    }
}

// selective activation (R36): a leaf's own samples -- "excluding those used for
// filtering", the overlap copies -- are the samples whose own key descends to it
__global__ void k_leaf_own(const mpg_guide_sample *rec, int64_t n, const int4 *nodes, int root_ref, int *leaf_own) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const mpg_guide_sample r = rec[i];
        if (!gs_valid(r)) continue;
        int ref = root_ref;
        while (ref >= 0) {
            const int4 nd = __ldg(nodes + ref);
            ref = gs_key(r, nd.y) < __int_as_float(nd.x) ? nd.z : nd.w;
        }
        atomicAdd(leaf_own + ~ref, 1);
    }
}

// per (leaf, type): E_tau (fp64, group order) and the integer lobe weights' prefix (R30)
__global__ void k_group_tables(const mpg_guide_sample *rec, const int *lobe_sample, const int *grp_off, int n_leaves,
                               double *E, unsigned long long *lobe_prefix) {
    int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n_leaves * 126) return;
    int l = id / 126, t = id % 126;
    int glo = grp_off[l * 127 + t], ghi = grp_off[l * 127 + t + 1];
    double e = 0.0;
    float wmax = 0.0f;
    for (int q = glo; q < ghi; q++) {
        float w = rec[lobe_sample[q]].w;
        e = __dadd_rn(e, (double)w);
        wmax = fmaxf(wmax, w);
    }
    E[(size_t)l * 126 + t] = e;
    unsigned long long acc = 0;
    for (int q = glo; q < ghi; q++) {
        float w = rec[lobe_sample[q]].w;
        unsigned long long W = (unsigned long long)floorf(FM(FD(w, wmax), 1048576.0f));
        if (W < 1ull) W = 1ull;
        acc += W;
        lobe_prefix[q] = acc;
    }
}

// glossy separator lobe (Eq. 14, R35): GGX(alpha) D(h) / (4 cos_v cos_D), fp32 as the oracle
__device__ __forceinline__ float separator_rho(float4 n, float4 wv, float ox, float oy, float oz, float alpha) {
    float cv = FA(FA(FM(n.x, wv.x), FM(n.y, wv.y)), FM(n.z, wv.z));
    float cl = FA(FA(FM(n.x, ox), FM(n.y, oy)), FM(n.z, oz));
    if (!(cv > 0.0f) || !(cl > 0.0f)) return 0.0f;
    float hx = FA(wv.x, ox), hy = FA(wv.y, oy), hz = FA(wv.z, oz);
    float hl = __fsqrt_rn(FA(FA(FM(hx, hx), FM(hy, hy)), FM(hz, hz)));
    hx = FD(hx, hl); hy = FD(hy, hl); hz = FD(hz, hl);
    float nh = FA(FA(FM(n.x, hx), FM(n.y, hy)), FM(n.z, hz));
    float a2 = FM(alpha, alpha);
    float t = FA(FM(FM(nh, nh), FS(a2, 1.0f)), 1.0f);
    float D = FD(a2, FM(3.14159265358979323846f, FM(t, t)));
    return FD(D, FM(FM(4.0f, cv), cl));
}

// sample records of one walk call (Eq. 9 samples; mirrors orc_record_samples)
__global__ void k_record(mpg_guide_sample *out, const float4 *xD, int spp, const float4 *xL, const float4 *chain0,
                         const uint8_t *status, const float *w, const uint16_t *ctype, int64_t n, const float4 *sep_wv,
                         const float4 *sep_n, float sep_alpha) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        mpg_guide_sample r;
        float4 d = xD[i / spp], l = xL[i];
        r.xD[0] = d.x; r.xD[1] = d.y; r.xD[2] = d.z;
        r.xL[0] = l.x; r.xL[1] = l.y; r.xL[2] = l.z;
        r.omega[0] = r.omega[1] = r.omega[2] = 0.0f;
        r.w = 0.0f;
        r.type = -1;
        r.pad = 0;
        uint32_t ct = ctype[i];
        int kk = (int)(ct & 15u);
        if (status[i] == 0 && w[i] > 0.0f && kk >= 1 && kk <= 6) {
            float4 x1 = chain0[i];
            float dx = FS(x1.x, d.x), dy = FS(x1.y, d.y), dz = FS(x1.z, d.z);
            float ln = __fsqrt_rn(FA(FA(FM(dx, dx), FM(dy, dy)), FM(dz, dz)));
            r.omega[0] = FD(dx, ln); r.omega[1] = FD(dy, ln); r.omega[2] = FD(dz, ln);
            r.type = (1 << kk) - 2 + (int)(ct >> 4);
            r.w = w[i];
            if (sep_wv) { // glossy separator: product weighting (Eq. 14)
                r.w = FM(w[i], separator_rho(sep_n[i / spp], sep_wv[i / spp], r.omega[0], r.omega[1], r.omega[2],
                                             sep_alpha));
                if (!(r.w > 0.0f)) { r.w = 0.0f; r.type = -1; r.omega[0] = r.omega[1] = r.omega[2] = 0.0f; }
            }
        }
        out[i] = r;
    }
}

#define ST_TRY(expr)                                                                                    \
    do {                                                                                                \
        cudaError_t e_ = (expr);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? MPG_ERR_OOM : MPG_ERR_CUDA,                   \
                        std::string("stree build: ") + #expr + ": " + cudaGetErrorString(e_));          \
    } while (0)

struct HNode {
    int64_t b, n;
    float lo[6], hi[6];
    int depth, parent, side;
};

static inline float host_o2f(unsigned u) {
    unsigned v = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &v, 4);
    return f;
}

// MPG_STREE_PROFILE=1: per-phase wall times of the build (synchronising after each phase), on stderr
struct StreeProf {
    bool on = getenv("MPG_STREE_PROFILE") != nullptr;
    std::vector<std::pair<std::string, double>> acc;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *phase, cudaStream_t st) {
        if (!on) return;
        cudaStreamSynchronize(st);
        auto now = std::chrono::steady_clock::now();
        double ms = std::chrono::duration<double, std::milli>(now - t).count();
        t = now;
        for (auto &a : acc)
            if (a.first == phase) { a.second += ms; return; }
        acc.emplace_back(phase, ms);
    }
    ~StreeProf() {
        if (!on) return;
        double tot = 0;
        for (auto &a : acc) tot += a.second;
        fprintf(stderr, "stree_build %.3f ms:", tot);
        for (auto &a : acc) fprintf(stderr, " %s=%.3f", a.first.c_str(), a.second);
        fprintf(stderr, "\n");
    }
};

// Build the tree and tables from the recorded samples (R28-R31); synchronous on st.
static mpg_status stree_build(StreeState *T, cudaStream_t st) {
    StreeProf prof;
    prof.mark("start", st);
    const int64_t n = T->n_rec;
    const int nsm = 148;
    // 1. sample ids (record order) and the root box
    ST_TRY(T->flags.reserve(n));
    ST_TRY(T->ids_a.reserve(n));
    ST_TRY(T->bbox.reserve(12));
    ST_TRY(T->nv.reserve(1));
    unsigned init[12];
    for (int a = 0; a < 6; a++) { init[a] = 0xffffffffu; init[6 + a] = 0u; }
    ST_TRY(cudaMemcpyAsync(T->bbox.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    int64_t nv = 0;
    unsigned bb[12];
    memcpy(bb, init, sizeof(bb));
    if (n > 0) {
        COUNT_LAUNCH(1);
        k_stree_valid<<<(int)std::min<int64_t>((n + 255) / 256, nsm * 8), 256, 0, st>>>(T->rec.p, n, T->flags.p,
                                                                                         T->bbox.p);
        ST_TRY(cudaPeekAtLastError());
        size_t tb = 0;
        thrust::counting_iterator<int> it(0);
        ST_TRY(cub::DeviceSelect::Flagged(nullptr, tb, it, T->flags.p, T->ids_a.p, T->nv.p, (int)n, st));
        ST_TRY(T->temp.reserve(tb));
        ST_TRY(cub::DeviceSelect::Flagged(T->temp.p, tb, it, T->flags.p, T->ids_a.p, T->nv.p, (int)n, st));
        int nvi = 0;
        ST_TRY(cudaMemcpyAsync(&nvi, T->nv.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        ST_TRY(cudaMemcpyAsync(bb, T->bbox.p, sizeof(bb), cudaMemcpyDeviceToHost, st));
        ST_TRY(cudaStreamSynchronize(st));
        nv = nvi;
    }
    prof.mark("select", st);
    T->n_valid = nv;
    double thr_d = floor((double)T->d.c_thr * sqrt((double)nv));
    T->thr = thr_d < 1.0 ? 1 : (int)thr_d;
    HNode root;
    root.b = 0;
    root.n = nv;
    for (int a = 0; a < 6; a++) {
        root.lo[a] = nv ? host_o2f(bb[a]) : 0.f;
        root.hi[a] = nv ? host_o2f(bb[6 + a]) : 0.f;
    }
    root.depth = 0;
    root.parent = -1;
    root.side = 0;
    int active[6], na = 0;
    for (int a = 0; a < 6; a++)
        if (nv > 0 && root.hi[a] > root.lo[a]) active[na++] = a;
    // 2. levels
    std::vector<HNode> level{root}, next;
    std::vector<int4> hnodes, segs;
    std::vector<int64_t> lb, lc;
    std::vector<int> split_idx;
    int64_t leaf_total = 0;
    ST_TRY(T->leaf_ids.reserve_keep((size_t)nv * 4, 0, st)); // overlap copies grow the lists (measured ~5x)
    int n_leaves = 0;
    int root_ref = ~0;
    int *cur = T->ids_a.p;
    bool cur_is_a = true;
    while (!level.empty()) {
        split_idx.clear();
        segs.clear();
        const int depth = level[0].depth;
        const int64_t leaf_prev = leaf_total;
        for (size_t i = 0; i < level.size(); i++) {
            HNode &nd = level[i];
            int ref;
            if (nd.n <= T->thr || nd.depth >= T->d.max_depth || na == 0) {
                ref = ~n_leaves++;
                lb.push_back(leaf_total);
                lc.push_back(nd.n);
                if (nd.n > 0) segs.push_back(make_int4((int)nd.b, (int)leaf_total, (int)nd.n, 0));
                leaf_total += nd.n;
            } else {
                ref = (int)hnodes.size();
                hnodes.push_back(make_int4(0, active[depth % std::max(na, 1)], 0, 0));
                split_idx.push_back((int)i);
            }
            if (nd.parent < 0) root_ref = ref;
            else if (nd.side == 0) hnodes[nd.parent].z = ref;
            else hnodes[nd.parent].w = ref;
        }
        ARG_CHECK(leaf_total < (1ll << 31) && n_leaves < (1 << 23), "STree too large (lobes >= 2^31 or leaves >= 2^23)");
        // one pinned upload per level: [leaf segments | level nodes (b, n) | split nodes (b, e) | (lo, hi)]
        const int n_ls = (int)segs.size(), nl = (int)level.size(), ns = (int)split_idx.size();
        const int a = ns ? active[depth % na] : 0;
        const size_t n4 = n_ls + (nl + 1) / 2 + (ns + 1) / 2 + (ns + 1) / 2;
        ST_TRY(T->hstage_a.reserve(n4));
        ST_TRY(T->dstage_a.reserve(n4));
        int4 *h4 = T->hstage_a.p;
        memcpy(h4, segs.data(), n_ls * sizeof(int4));
        // split nodes come first in the level array (children are laid out split-first):
        // only they are keyed and sorted
        int2 *h_lvl = (int2 *)(h4 + n_ls);
        for (int q = 0; q < ns; q++) h_lvl[q] = make_int2((int)level[split_idx[q]].b, (int)level[split_idx[q]].n);
        int2 *h_sbe = (int2 *)(h4 + n_ls + (nl + 1) / 2);
        float2 *h_lohi = (float2 *)(h4 + n_ls + (nl + 1) / 2 + (ns + 1) / 2);
        for (int q = 0; q < ns; q++) {
            const HNode &nd = level[split_idx[q]];
            h_sbe[q] = make_int2((int)nd.b, (int)(nd.b + nd.n));
            h_lohi[q] = make_float2(nd.lo[a], nd.hi[a]);
        }
        ST_TRY(cudaMemcpyAsync(T->dstage_a.p, h4, n4 * sizeof(int4), cudaMemcpyHostToDevice, st));
        const int4 *d_ls = T->dstage_a.p;
        const int2 *d_lvl = (const int2 *)(T->dstage_a.p + n_ls);
        const int2 *d_sbe = (const int2 *)(T->dstage_a.p + n_ls + (nl + 1) / 2);
        const float2 *d_lohi = (const float2 *)(T->dstage_a.p + n_ls + (nl + 1) / 2 + (ns + 1) / 2);
        if (n_ls) { // leaf lists of this level -> leaf_ids
            ST_TRY(T->leaf_ids.reserve_keep(leaf_total, leaf_prev, st));
            COUNT_LAUNCH(1);
            const int64_t ne = leaf_total - leaf_prev;
            k_copy_segments<<<(int)std::min<int64_t>((ne + 255) / 256, nsm * 8), 256, 0, st>>>(cur, T->leaf_ids.p, d_ls,
                                                                                              n_ls, ne);
            ST_TRY(cudaPeekAtLastError());
        }
        prof.mark("leafcopy", st);
        if (split_idx.empty()) break;
        int64_t n_cur = 0;   // elements of the split nodes: [0, n_cur) of the level array
        for (int q = 0; q < ns; q++) n_cur = std::max<int64_t>(n_cur, level[split_idx[q]].b + level[split_idx[q]].n);
        ST_TRY(T->keys_a.reserve(n_cur));
        ST_TRY(T->keys_b.reserve(n_cur));
        ST_TRY(T->split_out.reserve(2 * ns));
        ST_TRY(T->hsplit.reserve(2 * ns));
        DBuf<int> &sorted_ids = T->ids_c; // this level's ids, each node's list sorted
        ST_TRY(sorted_ids.reserve(n_cur));
        COUNT_LAUNCH(1);
        k_level_keys<<<(int)std::min<int64_t>((n_cur + 255) / 256, nsm * 8), 256, 0, st>>>(T->rec.p, cur, n_cur, d_lvl,
                                                                                            ns, a, T->keys_a.p);
        ST_TRY(cudaPeekAtLastError());
        prof.mark("keys", st);
        int nbits = 1;
        while ((1 << nbits) < ns) nbits++;
        size_t tb = 0;
        ST_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, T->keys_a.p, T->keys_b.p, cur, sorted_ids.p, (int)n_cur, 0,
                                               32 + nbits, st));
        ST_TRY(T->temp.reserve(tb));
        ST_TRY(cub::DeviceRadixSort::SortPairs(T->temp.p, tb, T->keys_a.p, T->keys_b.p, cur, sorted_ids.p, (int)n_cur,
                                               0, 32 + nbits, st));
        prof.mark("sort", st);
        COUNT_LAUNCH(1);
        k_stree_split<<<(ns + 127) / 128, 128, 0, st>>>(T->keys_b.p, d_sbe, d_lohi, ns, T->d.eps, T->split_out.p);
        ST_TRY(cudaPeekAtLastError());
        ST_TRY(cudaMemcpyAsync(T->hsplit.p, T->split_out.p, 2 * ns * sizeof(int4), cudaMemcpyDeviceToHost, st));
        ST_TRY(cudaStreamSynchronize(st));
        const int4 *so = T->hsplit.p;
        prof.mark("split", st);
        next.clear();
        segs.clear();
        int64_t off = 0;
        int node_id = (int)hnodes.size() - ns;
        for (int q = 0; q < ns; q++, node_id++) {
            const HNode &nd = level[split_idx[q]];
            int m = so[2 * q].x, eL = so[2 * q].y, eR = so[2 * q].z, s0 = so[2 * q].w, s1 = so[2 * q + 1].x;
            int cbits = so[2 * q + 1].y;
            float c;
            memcpy(&c, &cbits, 4);
            hnodes[node_id].x = cbits;
            for (int side = 0; side < 2; side++) {
                HNode ch = nd;
                int64_t b0 = side == 0 ? s0 : m - eL, b1 = side == 0 ? m + eR : s1;
                if (side == 0) ch.hi[a] = c;
                else ch.lo[a] = c;
                ch.b = nd.b + b0;   // source position in this level's sorted ids (laid out below)
                ch.n = b1 - b0;
                ch.depth = nd.depth + 1;
                ch.parent = node_id;
                ch.side = side;
                next.push_back(ch);
            }
        }
        // lay out the next level split-first (the children that will split, in order, then
        // the future leaves): the next level sorts only [0, split elements)
        for (int pass = 0; pass < 2; pass++) {
            for (auto &ch : next) {
                const bool will_leaf = ch.n <= T->thr || ch.depth >= T->d.max_depth || na == 0;
                if (will_leaf != (pass == 1)) continue;
                if (ch.n > 0) segs.push_back(make_int4((int)ch.b, (int)off, (int)ch.n, 0));
                ch.b = off;
                off += ch.n;
            }
        }
        ARG_CHECK(off < (1ll << 31), "STree level too large");
        DBuf<int> &dst = cur_is_a ? T->ids_b : T->ids_a;
        ST_TRY(dst.reserve(off));
        if (!segs.empty()) {
            ST_TRY(T->hstage_b.reserve(segs.size()));
            ST_TRY(T->dstage_b.reserve(segs.size()));
            memcpy(T->hstage_b.p, segs.data(), segs.size() * sizeof(int4));
            ST_TRY(cudaMemcpyAsync(T->dstage_b.p, T->hstage_b.p, segs.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
            COUNT_LAUNCH(1);
            k_copy_segments<<<(int)std::min<int64_t>((off + 255) / 256, nsm * 8), 256, 0, st>>>(
                sorted_ids.p, dst.p, T->dstage_b.p, (int)segs.size(), off);
            ST_TRY(cudaPeekAtLastError());
        }
        prof.mark("childcopy", st);
        cur = dst.p;
        cur_is_a = !cur_is_a;
        level.swap(next);
    }
    // 3. tree upload
    T->root_ref = root_ref;
    T->n_nodes = (int)hnodes.size();
    T->n_leaves = n_leaves;
    T->n_lobes = leaf_total;
    ST_TRY(T->nodes.reserve(hnodes.size()));
    ST_TRY(T->leaf_begin.reserve(n_leaves));
    ST_TRY(T->leaf_count.reserve(n_leaves));
    if (!hnodes.empty())
        ST_TRY(cudaMemcpyAsync(T->nodes.p, hnodes.data(), hnodes.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    ST_TRY(cudaMemcpyAsync(T->leaf_begin.p, lb.data(), n_leaves * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    ST_TRY(cudaMemcpyAsync(T->leaf_count.p, lc.data(), n_leaves * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    prof.mark("upload", st);
    // 4. lobes grouped by (leaf, type), stable within the leaf's list
    const int64_t NL = leaf_total;
    ST_TRY(T->grp_off.reserve((size_t)n_leaves * 127));
    ST_TRY(T->E.reserve((size_t)n_leaves * 126));
    ST_TRY(T->n_prefix.reserve((size_t)n_leaves * 6));
    ST_TRY(T->type_prefix.reserve((size_t)n_leaves * 126));
    ST_TRY(T->lobe_sample.reserve(NL));
    ST_TRY(T->lobe_prefix.reserve(NL));
    ST_TRY(T->lobe_mu.reserve(NL));
    ST_TRY(T->keys_a.reserve(NL));
    ST_TRY(T->keys_b.reserve(NL));
    if (NL > 0) {
        COUNT_LAUNCH(1);
        k_lobe_keys<<<n_leaves, 128, 0, st>>>(T->rec.p, T->leaf_ids.p, T->leaf_begin.p, T->leaf_count.p, T->keys_a.p);
        ST_TRY(cudaPeekAtLastError());
        int lbits = 1;
        while ((1 << lbits) < n_leaves) lbits++;
        size_t tb = 0;
        ST_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, T->keys_a.p, T->keys_b.p, (int)NL, 0, 40 + lbits, st));
        ST_TRY(T->temp.reserve(tb));
        ST_TRY(cub::DeviceRadixSort::SortKeys(T->temp.p, tb, T->keys_a.p, T->keys_b.p, (int)NL, 0, 40 + lbits, st));
        int blocks = (int)std::min<int64_t>((NL + 255) / 256, nsm * 8);
        COUNT_LAUNCH(1);
        k_lobe_sample<<<blocks, 256, 0, st>>>(T->keys_b.p, T->leaf_ids.p, NL, T->lobe_sample.p);
        ST_TRY(cudaPeekAtLastError());
    }
    prof.mark("lobesort", st);
    COUNT_LAUNCH(1);
    k_grp_off<<<(n_leaves * 127 + 255) / 256, 256, 0, st>>>(T->keys_b.p, NL, n_leaves, T->grp_off.p);
    ST_TRY(cudaPeekAtLastError());
    if (NL > 0) {
        COUNT_LAUNCH(1);
        k_lobe_kappa<<<(int)std::min<int64_t>((NL + 127) / 128, nsm * 16), 128, 0, st>>>(
            T->rec.p, T->keys_b.p, T->lobe_sample.p, T->grp_off.p, NL, T->d.kappa_min, T->d.kappa_max, T->lobe_mu.p);
        ST_TRY(cudaPeekAtLastError());
    }
    prof.mark("kappa", st);
    COUNT_LAUNCH(1);
    k_group_tables<<<(n_leaves * 126 + 127) / 128, 128, 0, st>>>(T->rec.p, T->lobe_sample.p, T->grp_off.p, n_leaves,
                                                                  T->E.p, T->lobe_prefix.p);
    ST_TRY(cudaPeekAtLastError());
    prof.mark("groups", st);
    COUNT_LAUNCH(1);
    k_dir_cell_tables<<<(n_leaves + 127) / 128, 128, 0, st>>>(T->E.p, n_leaves, T->n_prefix.p, T->type_prefix.p);
    ST_TRY(cudaPeekAtLastError());
    ST_TRY(T->leaf_own.reserve(std::max(n_leaves, 1)));
    ST_TRY(cudaMemsetAsync(T->leaf_own.p, 0, sizeof(int) * std::max(n_leaves, 1), st));
    if (T->n_rec > 0) {
        COUNT_LAUNCH(1);
        k_leaf_own<<<(int)std::min<int64_t>((T->n_rec + 255) / 256, nsm * 8), 256, 0, st>>>(
            T->rec.p, T->n_rec, T->nodes.p, T->root_ref, T->leaf_own.p);
        ST_TRY(cudaPeekAtLastError());
    }
    ST_TRY(cudaStreamSynchronize(st));
    prof.mark("tables", st);
    if (!T->d.keep_all) T->n_rec = 0; // "last iteration only" (P:426 footnote) unless keep_all
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_create_stree(const mpg_stree_desc *desc, mpg_guide **out) {
    ARG_CHECK(desc && out, "NULL argument");
    ARG_CHECK(desc->max_samples >= 0 && desc->max_samples < (1ll << 31), "max_samples must be in [0, 2^31)");
    ARG_CHECK(desc->eps >= 0.f && desc->eps < 0.5f, "eps must be in [0, 0.5)");
    ARG_CHECK(desc->c_thr > 0.f, "c_thr must be > 0");
    ARG_CHECK(desc->kappa_min >= 0.f && desc->kappa_max >= desc->kappa_min, "bad kappa clamp");
    ARG_CHECK(desc->max_depth >= 0 && desc->max_depth <= 64, "max_depth must be in [0, 64]");
    mpg_guide *g = new mpg_guide();
    memset(&g->desc, 0, sizeof(g->desc));
    g->desc.domain = 2;
    g->desc.n_types = 126;
    g->n_types = 126;
    g->stree = new StreeState();
    g->stree->d = *desc;
    // pre-size the build's buffers for max_samples (measured: ~22 % of records are samples on
    // configs[4], lobes ~5x the samples, a level ~1.2x its parent): growth inside a rebuild
    // costs cudaMalloc/cudaFree device syncs (~1 s on the first full-size rebuild otherwise)
    StreeState *T0 = g->stree;
    const size_t ms = (size_t)std::max<int64_t>(desc->max_samples, 1);
    bool okr = T0->flags.reserve(ms) == cudaSuccess && T0->ids_a.reserve(ms) == cudaSuccess &&
               T0->ids_b.reserve(ms) == cudaSuccess && T0->ids_c.reserve(ms) == cudaSuccess &&
               T0->keys_a.reserve(ms * 3 / 2) == cudaSuccess && T0->keys_b.reserve(ms * 3 / 2) == cudaSuccess &&
               T0->leaf_ids.reserve(ms * 3 / 2) == cudaSuccess && T0->lobe_sample.reserve(ms * 3 / 2) == cudaSuccess &&
               T0->lobe_prefix.reserve(ms * 3 / 2) == cudaSuccess && T0->lobe_mu.reserve(ms * 3 / 2) == cudaSuccess;
    if (!okr || g->stree->rec.reserve(desc->max_samples) != cudaSuccess) {
        mpg_guide_destroy(g);
        return fail(MPG_ERR_OOM, "STree sample buffer allocation failed");
    }
    cudaStream_t s0 = 0;
    mpg_status st = stree_build(g->stree, s0); // empty tree
    if (st != MPG_OK) {
        mpg_guide_destroy(g);
        return st;
    }
    g->ready = true;
    *out = g;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_record_samples(mpg_guide *g, const mpg_query *q, const mpg_seed_buf *sb,
                                               const mpg_walk_buf *wb, int64_t n, void *stream) {
    ARG_CHECK(g && g->stree && q && sb && wb, "needs an STree guide and query/seeds/walks");
    ARG_CHECK(q->xD && sb->xL && wb->chain && wb->status && wb->w && wb->ctype, "NULL array");
    ARG_CHECK(q->spp >= 1 && n == q->n_recv * q->spp, "n must equal n_recv*spp");
    StreeState *T = g->stree;
    ARG_CHECK(T->n_rec + n <= T->d.max_samples, "STree sample buffer full (max_samples)");
    if (n == 0) return MPG_OK;
    COUNT_LAUNCH(1);
    k_record<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, as_stream(stream)>>>(
        T->rec.p + T->n_rec, (const float4 *)q->xD, q->spp, (const float4 *)sb->xL, (const float4 *)wb->chain,
        wb->status, wb->w, wb->ctype, n, T->sep_wv, T->sep_n, T->sep_alpha);
    CUDA_TRY(cudaPeekAtLastError());
    T->n_rec += n;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_set_separator(mpg_guide *g, const float *wv, const float *nD, float alpha) {
    ARG_CHECK(g && g->stree, "needs an STree guide");
    ARG_CHECK((wv == nullptr) == (nD == nullptr), "wv and nD together");
    ARG_CHECK(!wv || (alpha > 0.f && alpha <= 1.f), "GGX alpha in (0, 1]");
    g->stree->sep_wv = (const float4 *)wv;
    g->stree->sep_n = (const float4 *)nD;
    g->stree->sep_alpha = alpha;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_set_samples(mpg_guide *g, const mpg_guide_sample *records, int64_t n, void *stream) {
    ARG_CHECK(g && g->stree && (records || n == 0), "needs an STree guide and records");
    ARG_CHECK(n >= 0 && n <= g->stree->d.max_samples, "n exceeds max_samples");
    if (n) CUDA_TRY(cudaMemcpyAsync(g->stree->rec.p, records, n * sizeof(mpg_guide_sample), cudaMemcpyDeviceToDevice,
                                    as_stream(stream)));
    g->stree->n_rec = n;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_get_samples(const mpg_guide *g, mpg_guide_sample *records, int64_t *n, void *stream) {
    ARG_CHECK(g && g->stree && n, "needs an STree guide and n");
    int64_t have = g->stree->n_rec;
    if (records) {
        ARG_CHECK(*n >= have, "records capacity too small");
        if (have) CUDA_TRY(cudaMemcpyAsync(records, g->stree->rec.p, have * sizeof(mpg_guide_sample),
                                           cudaMemcpyDeviceToDevice, as_stream(stream)));
    }
    *n = have;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_stree_info(const mpg_guide *g, mpg_stree_info *info) {
    ARG_CHECK(g && g->stree && info, "needs an STree guide");
    const StreeState *T = g->stree;
    info->n_nodes = T->n_nodes;
    info->n_leaves = T->n_leaves;
    info->root_ref = T->root_ref;
    info->thr = T->thr;
    info->n_valid = T->n_valid;
    info->n_lobes = T->n_lobes;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_download_stree(const mpg_guide *g, int32_t *nodes, int64_t *leaf_begin,
                                               int64_t *leaf_count, int32_t *leaf_ids, int32_t *grp_off,
                                               int32_t *lobe_sample, uint64_t *lobe_prefix, float *lobe_mu,
                                               uint64_t *n_prefix, uint64_t *type_prefix, int32_t *leaf_own,
                                               void *stream) {
    ARG_CHECK(g && g->stree, "needs an STree guide");
    const StreeState *T = g->stree;
    cudaStream_t s = as_stream(stream);
    const cudaMemcpyKind K = cudaMemcpyDeviceToDevice;
    const size_t L = (size_t)T->n_leaves, NL = (size_t)T->n_lobes;
    if (nodes && T->n_nodes) CUDA_TRY(cudaMemcpyAsync(nodes, T->nodes.p, T->n_nodes * sizeof(int4), K, s));
    if (leaf_begin) CUDA_TRY(cudaMemcpyAsync(leaf_begin, T->leaf_begin.p, L * 8, K, s));
    if (leaf_count) CUDA_TRY(cudaMemcpyAsync(leaf_count, T->leaf_count.p, L * 8, K, s));
    if (leaf_ids && NL) CUDA_TRY(cudaMemcpyAsync(leaf_ids, T->leaf_ids.p, NL * 4, K, s));
    if (grp_off) CUDA_TRY(cudaMemcpyAsync(grp_off, T->grp_off.p, L * 127 * 4, K, s));
    if (lobe_sample && NL) CUDA_TRY(cudaMemcpyAsync(lobe_sample, T->lobe_sample.p, NL * 4, K, s));
    if (lobe_prefix && NL) CUDA_TRY(cudaMemcpyAsync(lobe_prefix, T->lobe_prefix.p, NL * 8, K, s));
    if (lobe_mu && NL) CUDA_TRY(cudaMemcpyAsync(lobe_mu, T->lobe_mu.p, NL * 16, K, s));
    if (n_prefix) CUDA_TRY(cudaMemcpyAsync(n_prefix, T->n_prefix.p, L * 6 * 8, K, s));
    if (type_prefix) CUDA_TRY(cudaMemcpyAsync(type_prefix, T->type_prefix.p, L * 126 * 8, K, s));
    if (leaf_own && L) CUDA_TRY(cudaMemcpyAsync(leaf_own, T->leaf_own.p, L * 4, K, s));
    return MPG_OK;
}

static void stree_clear(StreeState *T) { T->n_rec = 0; }
