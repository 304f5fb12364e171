// mpg.cu -- libmpg.so: the C ABI of include/mpg.h, host-side scene/BVH build,
// guide tables, and the launch of the sm_100a kernels (seed, walk, estimate,
// guide build/accumulate, debug trace).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared
//        -Xcompiler -fPIC -I include (see paper_2311_12818_b200/build.py)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <atomic>
#include <functional>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "mpg.h"
#include "device_common.cuh"
#include "seed.cuh"
#include "walk.cuh"

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};   // mpg_kernel_launches()
#define COUNT_LAUNCH(n) g_launches.fetch_add((n), std::memory_order_relaxed)
static mpg_status fail(mpg_status s, const std::string &msg) {
    g_err = msg;
    return s;
}
#define CUDA_TRY(expr)                                                                                  \
    do {                                                                                                \
        cudaError_t e_ = (expr);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? MPG_ERR_OOM : MPG_ERR_CUDA,                   \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                           \
    } while (0)
#define ARG_CHECK(cond, msg)                                                                            \
    do {                                                                                                \
        if (!(cond)) return fail(MPG_ERR_INVALID_ARG, msg);                                             \
    } while (0)

static cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ----------------------------------------------------------------------------
// opaque objects
// ----------------------------------------------------------------------------
struct mpg_scene {
    DScene d;
    std::vector<void *> allocs;
    size_t bytes = 0;
    size_t trav_bytes = 0;  // nodes + triangle positions, contiguous from d.nodes
    int n_vert = 0;
    bool glossy = false;    // a surface has roughness > 0: the walk runs the glossy kernels (R37)
};

struct StreeState;
static void stree_state_free(StreeState *t);
struct mpg_guide {
    mpg_guide_desc desc;
    StreeState *stree = nullptr;  // domain 2: STree + vMF guide (stree.cuh)
    int n_cells = 0, n_bins = 0, n_types = 1;
    uint64_t *prefix = nullptr;   // domain 0: [cells][bins]
    float *hist = nullptr;        // [cells][types][bins]
    // domain 1 (typed directions, R22)
    uint64_t *n_prefix = nullptr; // [cells][6]
    uint64_t *type_prefix = nullptr; // [cells][126]
    uint32_t *dir_prefix = nullptr;  // [cells][126][bins]
    double *type_energy = nullptr;   // scratch [cells][126]
    bool ready = false;
};

// ----------------------------------------------------------------------------
// host math
// ----------------------------------------------------------------------------
struct hv3 {
    double x, y, z;
};
static hv3 H(const float *f) { return {f[0], f[1], f[2]}; }
static hv3 hsub(hv3 a, hv3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
static hv3 hcross(hv3 a, hv3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
static double hlen(hv3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
static float3 F3(hv3 a) { return make_float3((float)a.x, (float)a.y, (float)a.z); }
static hv3 hnrm(hv3 a) {
    double l = hlen(a);
    return {a.x / l, a.y / l, a.z / l};
}

// ----------------------------------------------------------------------------
// binned-SAH BVH2 over all mesh triangles (host C++).  Node = two child boxes +
// two child refs (>= 0 inner node, < 0 leaf ~(start<<3 | count-1)), 64 bytes.
// ----------------------------------------------------------------------------
namespace {
struct BTri {
    float lo[3], hi[3], c[3];
};
struct BNode {
    float b[12];
    int c0, c1;
};
struct Builder {
    const std::vector<BTri> &T;
    std::vector<int> idx;
    std::vector<BNode> nodes;
    int max_depth = 0;
    // SAH: traversal cost relative to one triangle test; leaves of leaf_min..leaf_max
    // triangles (<= 8: the leaf ref holds count-1 in 3 bits).  MPG_SAH_CT /
    // MPG_LEAF_MIN / MPG_LEAF_MAX override for experiments.
    float sah_ct = 0.5f;
    int leaf_min = 2, leaf_max = 4;
    explicit Builder(const std::vector<BTri> &t) : T(t), idx(t.size()) {
        if (const char *v = getenv("MPG_SAH_CT")) sah_ct = (float)atof(v);
        if (const char *v = getenv("MPG_LEAF_MIN")) leaf_min = std::max(1, std::min(8, atoi(v)));
        if (const char *v = getenv("MPG_LEAF_MAX")) leaf_max = std::max(leaf_min, std::min(8, atoi(v)));
        for (size_t i = 0; i < t.size(); i++) idx[i] = (int)i;
    }
    static float area(const float lo[3], const float hi[3]) {
        float dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        if (dx < 0 || dy < 0 || dz < 0) return 0.f;
        return 2.f * (dx * dy + dy * dz + dz * dx);
    }
    void bounds(int b, int e, float lo[3], float hi[3], float clo[3], float chi[3]) const {
        for (int a = 0; a < 3; a++) { lo[a] = clo[a] = 3e38f; hi[a] = chi[a] = -3e38f; }
        for (int i = b; i < e; i++) {
            const BTri &t = T[idx[i]];
            for (int a = 0; a < 3; a++) {
                lo[a] = std::min(lo[a], t.lo[a]); hi[a] = std::max(hi[a], t.hi[a]);
                clo[a] = std::min(clo[a], t.c[a]); chi[a] = std::max(chi[a], t.c[a]);
            }
        }
    }
    int leaf(int b, int e) { return ~((b << 3) | (e - b - 1)); }
    // returns child ref; box of the range in lo/hi
    int build(int b, int e, int depth, float lo[3], float hi[3]) {
        max_depth = std::max(max_depth, depth);
        float clo[3], chi[3];
        bounds(b, e, lo, hi, clo, chi);
        int n = e - b;
        if (n <= leaf_min) return leaf(b, e);
        const int NB = 32;
        int best_axis = -1, best_split = -1;
        float best_cost = 3e38f;
        if (depth < 56) {
            for (int a = 0; a < 3; a++) {
                float ext = chi[a] - clo[a];
                if (!(ext > 0.f)) continue;
                int cnt[NB] = {0};
                float blo[NB][3], bhi[NB][3];
                for (int j = 0; j < NB; j++)
                    for (int c = 0; c < 3; c++) { blo[j][c] = 3e38f; bhi[j][c] = -3e38f; }
                float sc = NB / ext;
                for (int i = b; i < e; i++) {
                    const BTri &t = T[idx[i]];
                    int j = std::min(NB - 1, (int)((t.c[a] - clo[a]) * sc));
                    cnt[j]++;
                    for (int c = 0; c < 3; c++) { blo[j][c] = std::min(blo[j][c], t.lo[c]); bhi[j][c] = std::max(bhi[j][c], t.hi[c]); }
                }
                float rA[NB];
                int rN[NB];
                float alo[3] = {3e38f, 3e38f, 3e38f}, ahi[3] = {-3e38f, -3e38f, -3e38f};
                int acc = 0;
                for (int j = NB - 1; j > 0; j--) {
                    for (int c = 0; c < 3; c++) { alo[c] = std::min(alo[c], blo[j][c]); ahi[c] = std::max(ahi[c], bhi[j][c]); }
                    acc += cnt[j];
                    rA[j] = area(alo, ahi);
                    rN[j] = acc;
                }
                for (int c = 0; c < 3; c++) { alo[c] = 3e38f; ahi[c] = -3e38f; }
                acc = 0;
                for (int j = 0; j < NB - 1; j++) {
                    for (int c = 0; c < 3; c++) { alo[c] = std::min(alo[c], blo[j][c]); ahi[c] = std::max(ahi[c], bhi[j][c]); }
                    acc += cnt[j];
                    if (acc == 0 || rN[j + 1] == 0) continue;
                    float cost = area(alo, ahi) * acc + rA[j + 1] * rN[j + 1];
                    if (cost < best_cost) { best_cost = cost; best_axis = a; best_split = j; }
                }
            }
        }
        float pa = area(lo, hi);
        float leaf_cost = (float)n;
        float split_cost = sah_ct + (pa > 0.f ? best_cost / pa : 3e38f);
        if (n <= leaf_max && (best_axis < 0 || split_cost >= leaf_cost)) return leaf(b, e);
        int mid;
        if (best_axis >= 0) {
            float ext = chi[best_axis] - clo[best_axis], sc = NB / ext, c0 = clo[best_axis];
            int a = best_axis, s = best_split;
            mid = (int)(std::partition(idx.begin() + b, idx.begin() + e, [&](int t) {
                        return std::min(NB - 1, (int)((T[t].c[a] - c0) * sc)) <= s;
                    }) - idx.begin());
            if (mid == b || mid == e) mid = (b + e) / 2;
        } else {
            int a = 0;
            for (int c = 1; c < 3; c++) if (chi[c] - clo[c] > chi[a] - clo[a]) a = c;
            mid = (b + e) / 2;
            std::nth_element(idx.begin() + b, idx.begin() + mid, idx.begin() + e,
                             [&](int x, int y) { return T[x].c[a] < T[y].c[a]; });
        }
        int id = (int)nodes.size();
        nodes.push_back(BNode());
        float l0[3], h0[3], l1[3], h1[3];
        int c0 = build(b, mid, depth + 1, l0, h0);
        int c1 = build(mid, e, depth + 1, l1, h1);
        BNode &nd = nodes[id];
        nd.b[0] = l0[0]; nd.b[1] = l0[1]; nd.b[2] = l0[2]; nd.b[3] = h0[0];
        nd.b[4] = h0[1]; nd.b[5] = h0[2]; nd.b[6] = l1[0]; nd.b[7] = l1[1];
        nd.b[8] = l1[2]; nd.b[9] = h1[0]; nd.b[10] = h1[1]; nd.b[11] = h1[2];
        nd.c0 = c0; nd.c1 = c1;
        return id;
    }
};
} // namespace

template <class T>
static mpg_status upload(mpg_scene *s, const std::vector<T> &v, const T **dst) {
    void *p = nullptr;
    size_t bytes = std::max<size_t>(sizeof(T), v.size() * sizeof(T));
    CUDA_TRY(cudaMalloc(&p, bytes));
    s->allocs.push_back(p);
    s->bytes += bytes;
    if (!v.empty()) CUDA_TRY(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    *dst = reinterpret_cast<const T *>(p);
    return MPG_OK;
}

extern "C" mpg_status mpg_scene_destroy(mpg_scene *scene) {
    if (!scene) return MPG_OK;
    for (void *p : scene->allocs) cudaFree(p);
    delete scene;
    return MPG_OK;
}

extern "C" mpg_status mpg_scene_create(const mpg_surface_desc *surfaces, int32_t n_surf, const mpg_light_desc *lights,
                                       int32_t n_light, void *stream, mpg_scene **out) {
    (void)stream;
    ARG_CHECK(out, "out is NULL");
    *out = nullptr;
    ARG_CHECK(surfaces && n_surf >= 1 && n_surf <= DS_MAX_SURF, "need 1..16 surfaces");
    ARG_CHECK(lights && n_light >= 1 && n_light <= DS_MAX_LIGHT, "need 1..8 lights");
    mpg_scene *s = new mpg_scene();
    memset(&s->d, 0, sizeof(DScene));
    DScene &d = s->d;
    d.n_surf = n_surf;
    d.n_light = n_light;
    // global triangle numbering: meshes concatenated in surface order
    std::vector<float4> vpos, vnrm;
    std::vector<int4> oidx;
    std::vector<int> tsurf;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    auto grow = [&](hv3 p) {
        double q[3] = {p.x, p.y, p.z};
        for (int a = 0; a < 3; a++) { lo[a] = std::min(lo[a], q[a]); hi[a] = std::max(hi[a], q[a]); }
    };
    for (int i = 0; i < n_surf; i++) {
        const mpg_surface_desc &sd = surfaces[i];
        DSurf &f = d.surf[i];
        if (sd.kind < 0 || sd.kind > 2 || sd.mat < 0 || sd.mat > 2) { mpg_scene_destroy(s); return fail(MPG_ERR_INVALID_ARG, "bad surface kind/mat"); }
        if (sd.mat == 1 && !(sd.eta_in > 0.f && sd.eta_out > 0.f && sd.eta_in != sd.eta_out)) {
            mpg_scene_destroy(s);
            return fail(MPG_ERR_INVALID_ARG, "dielectric needs eta_in != eta_out > 0 (R2: index-matched T excluded)");
        }
        f.kind = sd.kind; f.mat = sd.mat;
        f.eta_in = sd.eta_in > 0.f ? sd.eta_in : 1.f;
        f.eta_out = sd.eta_out > 0.f ? sd.eta_out : 1.f;
        f.refl = sd.reflectance;
        if (!(sd.roughness >= 0.f)) { mpg_scene_destroy(s); return fail(MPG_ERR_INVALID_ARG, "roughness must be >= 0"); }
        f.rough = sd.roughness;
        if (sd.roughness > 0.f) s->glossy = true;
        f.radius = sd.radius;
        f.center = F3(H(sd.center));
        f.origin = F3(H(sd.origin));
        f.eu = F3(H(sd.edge_u));
        f.ev = F3(H(sd.edge_v));
        f.nq = make_float3(0, 0, 1);
        if (sd.kind == 0) {
            if (!(sd.radius > 0.f)) { mpg_scene_destroy(s); return fail(MPG_ERR_INVALID_ARG, "sphere radius <= 0"); }
            hv3 c = H(sd.center);
            grow({c.x - sd.radius, c.y - sd.radius, c.z - sd.radius});
            grow({c.x + sd.radius, c.y + sd.radius, c.z + sd.radius});
        } else if (sd.kind == 1) {
            hv3 o = H(sd.origin), u = H(sd.edge_u), v = H(sd.edge_v);
            hv3 n = hcross(u, v);
            if (!(hlen(n) > 0)) { mpg_scene_destroy(s); return fail(MPG_ERR_INVALID_ARG, "degenerate quad"); }
            f.nq = F3(hnrm(n));
            grow(o); grow({o.x + u.x, o.y + u.y, o.z + u.z}); grow({o.x + v.x, o.y + v.y, o.z + v.z});
            grow({o.x + u.x + v.x, o.y + u.y + v.y, o.z + u.z + v.z});
        } else {
            if (!sd.positions || !sd.normals || !sd.indices || sd.n_vertices <= 0 || sd.n_triangles <= 0) {
                mpg_scene_destroy(s);
                return fail(MPG_ERR_INVALID_ARG, "mesh arrays missing");
            }
            int vb = (int)vpos.size();
            f.tri_begin = (int)oidx.size();
            f.tri_count = sd.n_triangles;
            for (int v = 0; v < sd.n_vertices; v++) {
                vpos.push_back(make_float4(sd.positions[3 * v], sd.positions[3 * v + 1], sd.positions[3 * v + 2], 0.f));
                vnrm.push_back(make_float4(sd.normals[3 * v], sd.normals[3 * v + 1], sd.normals[3 * v + 2], 0.f));
            }
            for (int t = 0; t < sd.n_triangles; t++) {
                int a = sd.indices[3 * t], b = sd.indices[3 * t + 1], c = sd.indices[3 * t + 2];
                if (a < 0 || b < 0 || c < 0 || a >= sd.n_vertices || b >= sd.n_vertices || c >= sd.n_vertices) {
                    mpg_scene_destroy(s);
                    return fail(MPG_ERR_INVALID_ARG, "mesh index out of range");
                }
                oidx.push_back(make_int4(vb + a, vb + b, vb + c, 0));
                tsurf.push_back(i);
                for (int q : {a, b, c}) grow(H(sd.positions + 3 * q));
            }
        }
    }
    d.n_tri = (int)oidx.size();
    for (int i = 0; i < n_light; i++) {
        const mpg_light_desc &ld = lights[i];
        DLight &L = d.light[i];
        ARG_CHECK(ld.kind == 0 || ld.kind == 1, "bad light kind");
        L.kind = ld.kind;
        L.emit = ld.emit;
        L.pos = F3(H(ld.position));
        L.eu = F3(H(ld.edge_u));
        L.ev = F3(H(ld.edge_v));
        hv3 c = H(ld.position);
        if (ld.kind == 1) {
            hv3 u = H(ld.edge_u), v = H(ld.edge_v), n = hcross(u, v);
            double area = hlen(n);
            if (!(area > 0)) { mpg_scene_destroy(s); return fail(MPG_ERR_INVALID_ARG, "degenerate area light"); }
            hv3 nn = hnrm(n), l1 = hnrm(u), l2 = hnrm(hcross(nn, l1));
            L.n = F3(nn); L.l1 = F3(l1); L.l2 = F3(l2);
            L.pdf = (float)(1.0 / (area * n_light));
            for (int sx = -1; sx <= 1; sx += 2)
                for (int sy = -1; sy <= 1; sy += 2)
                    grow({c.x + 0.5 * sx * u.x + 0.5 * sy * v.x, c.y + 0.5 * sx * u.y + 0.5 * sy * v.y,
                          c.z + 0.5 * sx * u.z + 0.5 * sy * v.z});
        } else {
            L.pdf = (float)(1.0 / n_light);
            L.n = make_float3(0, 0, 0);
            grow(c);
        }
    }
    d.extent = (float)std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                (hi[2] - lo[2]) * (hi[2] - lo[2]));
    // BVH
    std::vector<float4> nodes4, tpos, tnrm;
    d.bvh_w = 2;
    if (d.n_tri > 0) {
        std::vector<BTri> bt(d.n_tri);
        for (int t = 0; t < d.n_tri; t++) {
            const int4 &ix = oidx[t];
            const float4 *p[3] = {&vpos[ix.x], &vpos[ix.y], &vpos[ix.z]};
            for (int a = 0; a < 3; a++) {
                float v0 = (&p[0]->x)[a], v1 = (&p[1]->x)[a], v2 = (&p[2]->x)[a];
                bt[t].lo[a] = std::min(v0, std::min(v1, v2));
                bt[t].hi[a] = std::max(v0, std::max(v1, v2));
                bt[t].c[a] = (v0 + v1 + v2) * (1.0f / 3.0f);
            }
        }
        Builder B(bt);
        B.nodes.reserve(d.n_tri);
        float rlo[3], rhi[3];
        int root = B.build(0, d.n_tri, 0, rlo, rhi);
        if (root < 0) { // single leaf: wrap in a root with an empty sibling
            BNode nd;
            for (int a = 0; a < 3; a++) { nd.b[a] = rlo[a]; }
            nd.b[3] = rhi[0]; nd.b[4] = rhi[1]; nd.b[5] = rhi[2];
            for (int a = 6; a < 9; a++) nd.b[a] = 3e38f;
            for (int a = 9; a < 12; a++) nd.b[a] = 3e38f;   // empty sibling: point box at 3e38 (never entered)
            nd.c0 = root; nd.c1 = root;
            B.nodes.insert(B.nodes.begin(), nd);
        }
        if (B.max_depth > 60) { mpg_scene_destroy(s); return fail(MPG_ERR_UNSUPPORTED, "BVH too deep"); }
        {   // inflate child boxes by extent * 2^-20: keeps the FFMA slab test conservative (bvh_visit)
            const float e = d.extent * (1.0f / 1048576.0f);
            for (BNode &nd : B.nodes)
                for (int c = 0; c < 2; c++)
                    for (int a = 0; a < 3; a++) {
                        nd.b[6 * c + a] -= e;
                        nd.b[6 * c + 3 + a] += e;
                    }
        }
        int width = d.n_tri >= 65536 ? 4 : 2;
        if (const char *v = getenv("MPG_BVH_WIDTH")) width = atoi(v) == 4 ? 4 : 2;
        d.bvh_w = width;
        if (width == 4) {
        // collapse the binary SAH tree into a 4-wide one (children = grandchildren):
        // half the dependent node fetches per ray; 128-B SoA nodes (NODE_F4 float4)
        std::vector<float> w4;
        std::function<int(int)> collapse = [&](int n2) -> int {
            const BNode &nd = B.nodes[n2];
            int ref[4], cnt = 0;
            float box[4][6];
            for (int c = 0; c < 2; c++) {
                int ch = c == 0 ? nd.c0 : nd.c1;
                const float *bb = nd.b + 6 * c; // lo x,y,z, hi x,y,z
                if (ch >= 0) {
                    const BNode &g = B.nodes[ch];
                    for (int e = 0; e < 2; e++) {
                        ref[cnt] = e == 0 ? g.c0 : g.c1;
                        for (int a = 0; a < 6; a++) box[cnt][a] = g.b[6 * e + a];
                        cnt++;
                    }
                } else {
                    ref[cnt] = ch;
                    for (int a = 0; a < 6; a++) box[cnt][a] = bb[a];
                    cnt++;
                }
            }
            const int id = (int)(w4.size() / (4 * NODE_F4(4)));
            w4.resize(w4.size() + 4 * NODE_F4(4), 0.f);
            for (int j = 0; j < cnt; j++)
                if (ref[j] >= 0) ref[j] = collapse(ref[j]);
            float *o = w4.data() + (size_t)id * 4 * NODE_F4(4);
            for (int j = 0; j < 4; j++) {
                const bool on = j < cnt;
                for (int a = 0; a < 3; a++) {
                    // empty slot: a point box at (3e38, 3e38, 3e38) -- never entered for any
                    // direction sign (an inverted lo > hi box is NOT rejected by min/max slabs)
                    o[8 * a + j] = on ? box[j][a] : 3e38f;          // lo_a[j]
                    o[8 * a + 4 + j] = on ? box[j][3 + a] : 3e38f;  // hi_a[j]
                }
                int r = on ? ref[j] : 0x7fffffff;
                memcpy(&o[24 + j], &r, 4);
            }
            return id;
        };
        collapse(0);
        d.n_nodes = (int)(w4.size() / (4 * NODE_F4(4)));
        nodes4.resize((size_t)NODE_F4(4) * d.n_nodes);
        memcpy(nodes4.data(), w4.data(), w4.size() * sizeof(float));
        } else {
        d.n_nodes = (int)B.nodes.size();
        nodes4.resize(4 * d.n_nodes);
        for (int i = 0; i < d.n_nodes; i++) {
            const BNode &nd = B.nodes[i];
            nodes4[4 * i + 0] = make_float4(nd.b[0], nd.b[1], nd.b[2], nd.b[3]);
            nodes4[4 * i + 1] = make_float4(nd.b[4], nd.b[5], nd.b[6], nd.b[7]);
            nodes4[4 * i + 2] = make_float4(nd.b[8], nd.b[9], nd.b[10], nd.b[11]);
            int4 ch = make_int4(nd.c0, nd.c1, 0, 0);
            memcpy(&nodes4[4 * i + 3], &ch, sizeof(int4));
        }
        }
        {   // number the first levels breadth-first (root = 0, then its children, ...): the walk kernel can
            // stage nodes [0, MPG_TOP_NODES) in shared memory; the other nodes keep their relative order
            const int F4 = NODE_F4(width), NCH = width == 4 ? 4 : 2;
            auto child = [&](int n, int j) -> int & {
                return *reinterpret_cast<int *>(width == 4 ? &(&nodes4[(size_t)F4 * n + 6].x)[j] : &(&nodes4[(size_t)F4 * n + 3].x)[j]);
            };
            const int NB = std::min(d.n_nodes, 256);
            std::vector<int> order, newid(d.n_nodes, -1);
            order.push_back(0);
            for (size_t q = 0; q < order.size() && (int)order.size() < NB; q++)
                for (int j = 0; j < NCH && (int)order.size() < NB; j++) {
                    const int c = child(order[q], j);
                    if (c >= 0 && c != 0x7fffffff) order.push_back(c);
                }
            for (size_t q = 0; q < order.size(); q++) newid[order[q]] = (int)q;
            int nxt = (int)order.size();
            for (int n = 0; n < d.n_nodes; n++)
                if (newid[n] < 0) newid[n] = nxt++;
            std::vector<float4> re(nodes4.size());
            for (int n = 0; n < d.n_nodes; n++) {
                for (int j = 0; j < NCH; j++) {
                    int &c = child(n, j);
                    if (c >= 0 && c != 0x7fffffff) c = newid[c];
                }
                for (int f = 0; f < F4; f++) re[(size_t)F4 * newid[n] + f] = nodes4[(size_t)F4 * n + f];
            }
            nodes4.swap(re);
        }
        tpos.assign((size_t)TSTRIDE * d.n_tri, make_float4(0.f, 0.f, 0.f, 0.f));
        tnrm.resize(3 * d.n_tri);
        for (int j = 0; j < d.n_tri; j++) {
            int t = B.idx[j];
            int4 &ix = oidx[t];
            ix.w = j;
            int sid = tsurf[t];
            int spec = d.surf[sid].mat != 2 ? 1 : 0;
            float4 a = vpos[ix.x], b = vpos[ix.y], c = vpos[ix.z];
            int tw = t;
            memcpy(&a.w, &tw, 4);
            memcpy(&b.w, &sid, 4);
            memcpy(&c.w, &spec, 4);
            tpos[TSTRIDE * j] = a; tpos[TSTRIDE * j + 1] = b; tpos[TSTRIDE * j + 2] = c;
            tnrm[3 * j] = vnrm[ix.x]; tnrm[3 * j + 1] = vnrm[ix.y]; tnrm[3 * j + 2] = vnrm[ix.z];
        }
    }
    mpg_status st;
    // nodes and triangle positions (what traversal reads) in one allocation, so one L2
    // access-policy window can keep them resident against the walk's local-memory traffic
    {
        size_t nb = std::max<size_t>(1, nodes4.size()) * sizeof(float4), tb = std::max<size_t>(1, tpos.size()) * sizeof(float4);
        void *p = nullptr;
        cudaError_t e = cudaMalloc(&p, nb + tb);
        if (e != cudaSuccess) {
            mpg_scene_destroy(s);
            return fail(MPG_ERR_OOM, "scene allocation failed");
        }
        s->allocs.push_back(p);
        s->bytes += nb + tb;
        if (!nodes4.empty()) cudaMemcpy(p, nodes4.data(), nodes4.size() * sizeof(float4), cudaMemcpyHostToDevice);
        if (!tpos.empty()) cudaMemcpy((char *)p + nb, tpos.data(), tpos.size() * sizeof(float4), cudaMemcpyHostToDevice);
        d.nodes = (const float4 *)p;
        d.tpos = (const float4 *)((char *)p + nb);
        s->trav_bytes = nb + tb;
    }
    // edge adjacency in BVH order (refine_hit's fp64 triangle choice at shared edges, R17):
    // neighbour across the edge opposite vertex e of each triangle, -1 on a border
    std::vector<int4> tadj((size_t)d.n_tri, make_int4(-1, -1, -1, -1));
    {
        std::vector<std::pair<unsigned long long, int>> edges;   // (edge key, slot*4 + e)
        edges.reserve((size_t)3 * d.n_tri);
        for (int t = 0; t < d.n_tri; t++) {
            const int4 ix = oidx[t];
            const int v[3] = {ix.x, ix.y, ix.z};
            for (int e = 0; e < 3; e++) {
                unsigned long long p = (unsigned)v[(e + 1) % 3], q = (unsigned)v[(e + 2) % 3];
                if (p > q) std::swap(p, q);
                edges.push_back({(p << 32) | q, ix.w * 4 + e});
            }
        }
        std::sort(edges.begin(), edges.end());
        for (size_t i = 0; i + 1 < edges.size(); i++) {
            if (edges[i].first != edges[i + 1].first) continue;
            if (i + 2 < edges.size() && edges[i + 2].first == edges[i].first) {   // non-manifold edge: no link
                while (i + 1 < edges.size() && edges[i + 1].first == edges[i].first) i++;
                continue;
            }
            const int a = edges[i].second, b = edges[i + 1].second;
            (&tadj[a >> 2].x)[a & 3] = b >> 2;
            (&tadj[b >> 2].x)[b & 3] = a >> 2;
            i++;
        }
    }
    if ((st = upload(s, tnrm, &d.tnrm)) != MPG_OK || (st = upload(s, oidx, &d.oidx)) != MPG_OK ||
        (st = upload(s, vpos, &d.vpos)) != MPG_OK || (st = upload(s, tadj, &d.tadj)) != MPG_OK) {
        mpg_scene_destroy(s);
        return st;
    }
    s->n_vert = (int)vpos.size();
    *out = s;
    return MPG_OK;
}

extern "C" mpg_status mpg_scene_get_info(const mpg_scene *scene, mpg_scene_info *info) {
    ARG_CHECK(scene && info, "NULL argument");
    info->extent = scene->d.extent;
    info->n_surf = scene->d.n_surf;
    info->n_light = scene->d.n_light;
    info->n_tri = scene->d.n_tri;
    info->n_nodes = scene->d.n_nodes;
    info->bvh_width = scene->d.bvh_w;
    info->device_bytes = scene->bytes;
    return MPG_OK;
}

// ----------------------------------------------------------------------------
// debug trace kernel
// ----------------------------------------------------------------------------
template <int W>
__global__ void k_trace(const DScene S, const float4 *orig, const float4 *dir, int64_t n, float tmin, int spec_only,
                        float *t, int *prim, int *surf) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        LaneStats ls = {0, 0, 0};
        Hit h;
        ls.rays++;
        bool ok = trace<W>(S, xyz(orig[i]), nrmz(xyz(dir[i])), tmin, 3.0e38f, spec_only != 0, false, h, ls);
        t[i] = ok ? h.t : -1.0f;
        prim[i] = ok && h.prim >= 0 ? __float_as_int(S.tpos[TSTRIDE * h.prim].w) : -1;
        surf[i] = ok ? h.surf : -1;
    }
}

extern "C" mpg_status mpg_trace_rays(const mpg_scene *scene, const float *orig, const float *dir, int64_t n,
                                     float tmin, int32_t spec_only, float *t, int32_t *prim, int32_t *surf,
                                     void *stream) {
    ARG_CHECK(scene && orig && dir && t && prim && surf && n >= 0, "bad argument");
    if (n == 0) return MPG_OK;
    int blocks = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
    COUNT_LAUNCH(1);
    if (scene->d.bvh_w == 4)
        k_trace<4><<<blocks, 128, 0, as_stream(stream)>>>(scene->d, (const float4 *)orig, (const float4 *)dir, n, tmin,
                                                          spec_only, t, prim, surf);
    else
        k_trace<2><<<blocks, 128, 0, as_stream(stream)>>>(scene->d, (const float4 *)orig, (const float4 *)dir, n, tmin,
                                                          spec_only, t, prim, surf);
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}

// ----------------------------------------------------------------------------
// guide: integer defensive tables (R20), accumulate (Eq. 9), rebuild
// ----------------------------------------------------------------------------
#define GT_THREADS 256
__global__ void __launch_bounds__(GT_THREADS) k_guide_tables(const float *E, int nb, uint64_t *prefix) {
    __shared__ float s_max[GT_THREADS];
    __shared__ unsigned long long s_sum[GT_THREADS];
    const int c = blockIdx.x, tid = threadIdx.x;
    const float *e = E + (size_t)c * nb;
    uint64_t *pf = prefix + (size_t)c * nb;
    int per = (nb + GT_THREADS - 1) / GT_THREADS;
    int b0 = tid * per, b1 = min(nb, b0 + per);
    float m = 0.f;
    for (int b = b0; b < b1; b++) m = fmaxf(m, e[b]);
    s_max[tid] = m;
    __syncthreads();
    for (int o = GT_THREADS / 2; o > 0; o >>= 1) {
        if (tid < o) s_max[tid] = fmaxf(s_max[tid], s_max[tid + o]);
        __syncthreads();
    }
    float emax = s_max[0];
    auto Wb = [&](float eb) -> uint32_t {
        if (!(eb > 0.f) || !(emax > 0.f)) return 0u;
        uint32_t q = (uint32_t)floorf(__fmul_rn(__fdiv_rn(eb, emax), 1048576.0f));
        return q < 1u ? 1u : q;
    };
    unsigned long long loc = 0;
    for (int b = b0; b < b1; b++) loc += Wb(e[b]);
    s_sum[tid] = loc;
    __syncthreads();
    for (int o = GT_THREADS / 2; o > 0; o >>= 1) {
        if (tid < o) s_sum[tid] += s_sum[tid + o];
        __syncthreads();
    }
    unsigned long long sumW = s_sum[0];
    __syncthreads();
    auto Wp = [&](float eb) -> unsigned long long { return sumW == 0 ? 1ull : sumW + (unsigned long long)nb * Wb(eb); };
    loc = 0;
    for (int b = b0; b < b1; b++) loc += Wp(e[b]);
    s_sum[tid] = loc;
    __syncthreads();
    // inclusive Hillis-Steele scan over the per-thread totals
    for (int o = 1; o < GT_THREADS; o <<= 1) {
        unsigned long long v = tid >= o ? s_sum[tid - o] : 0ull;
        __syncthreads();
        s_sum[tid] += v;
        __syncthreads();
    }
    unsigned long long acc = tid > 0 ? s_sum[tid - 1] : 0ull;
    for (int b = b0; b < b1; b++) {
        acc += Wp(e[b]);
        pf[b] = acc;
    }
}

__global__ void k_fill_f32(float *p, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__device__ __forceinline__ int guide_cell(const mpg_guide_desc &g, float3 xD) {
    int cx = (int)floorf(FD(FM(FS(xD.x, g.grid_origin[0]), (float)g.cells_x), g.grid_extent[0]));
    int cz = (int)floorf(FD(FM(FS(xD.z, g.grid_origin[1]), (float)g.cells_y), g.grid_extent[1]));
    cx = min(max(cx, 0), g.cells_x - 1);
    cz = min(max(cz, 0), g.cells_y - 1);
    return cz * g.cells_x + cx;
}

// histogram[cell(x_D)][bin(x_1*)] += w (Eq. 9; lobes sit at the found chains),
// warp-aggregated: lanes with equal (cell,bin) keys combine before one atomic.
__global__ void k_accumulate(const mpg_guide_desc g, const float4 *xD, int spp, int64_t n, const float4 *chain0,
                             const uint8_t *status, const float *w, float *hist) {
    const int nb = g.bins_x * g.bins_y;
    const int lane = threadIdx.x & 31;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = base + threadIdx.x;
        int key = -1;
        float val = 0.f;
        if (i < n && status[i] == 0 && w[i] > 0.f) {
            float3 x1 = xyz(chain0[i]);
            int cell = guide_cell(g, xyz(xD[i / spp]));
            float u = (x1.x - g.uv_origin[0]) / g.uv_scale[0], v = (x1.z - g.uv_origin[1]) / g.uv_scale[1];
            int bx = min(max((int)floorf(u * g.bins_x), 0), g.bins_x - 1);
            int by = min(max((int)floorf(v * g.bins_y), 0), g.bins_y - 1);
            key = cell * nb + by * g.bins_x + bx;
            val = w[i];
        }
        unsigned grp = __match_any_sync(MPG_FULL, key);
        float sum = 0.f;
        for (int j = 0; j < 32; j++) {
            float vj = __shfl_sync(MPG_FULL, val, j);
            if (grp & (1u << j)) sum += vj;
        }
        if (key >= 0 && lane == __ffs(grp) - 1) atomicAdd(hist + key, sum);
    }
}

extern "C" mpg_status mpg_guide_create(const mpg_guide_desc *desc, mpg_guide **out) {
    ARG_CHECK(desc && out, "NULL argument");
    ARG_CHECK(desc->cells_x >= 1 && desc->cells_y >= 1 && desc->bins_x >= 1 && desc->bins_y >= 1, "empty guide");
    ARG_CHECK(desc->grid_extent[0] > 0.f && desc->grid_extent[1] > 0.f && desc->uv_scale[0] != 0.f &&
                  desc->uv_scale[1] != 0.f, "bad guide extents");
    ARG_CHECK((int64_t)desc->bins_x * desc->bins_y <= 65536, "at most 65536 bins per cell");
    ARG_CHECK(desc->domain == 0 || desc->domain == 1, "guide domain must be 0 (uv) or 1 (typed directions)");
    ARG_CHECK(desc->domain == 0 || desc->n_types == 126, "typed direction guide needs n_types = 126 (n <= 6)");
    mpg_guide *g = new mpg_guide();
    g->desc = *desc;
    g->n_cells = desc->cells_x * desc->cells_y;
    g->n_bins = desc->bins_x * desc->bins_y;
    g->n_types = desc->domain == 1 ? 126 : 1;
    size_t ne = (size_t)g->n_cells * g->n_types * g->n_bins;
    cudaError_t e = cudaMalloc(&g->hist, ne * sizeof(float));
    if (e == cudaSuccess) {
        if (desc->domain == 0) e = cudaMalloc(&g->prefix, ne * sizeof(uint64_t));
        else {
            e = cudaMalloc(&g->n_prefix, (size_t)g->n_cells * 6 * sizeof(uint64_t));
            if (e == cudaSuccess) e = cudaMalloc(&g->type_prefix, (size_t)g->n_cells * 126 * sizeof(uint64_t));
            if (e == cudaSuccess) e = cudaMalloc(&g->dir_prefix, ne * sizeof(uint32_t));
            if (e == cudaSuccess) e = cudaMalloc(&g->type_energy, (size_t)g->n_cells * 126 * sizeof(double));
        }
    }
    if (e != cudaSuccess) {
        mpg_guide_destroy(g);
        return fail(MPG_ERR_OOM, "guide allocation failed");
    }
    *out = g;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_destroy(mpg_guide *g) {
    if (!g) return MPG_OK;
    cudaFree(g->prefix);
    cudaFree(g->hist);
    cudaFree(g->n_prefix);
    cudaFree(g->type_prefix);
    cudaFree(g->dir_prefix);
    cudaFree(g->type_energy);
    stree_state_free(g->stree);
    delete g;
    return MPG_OK;
}

// ---- typed direction guide (configs[4], R22): tables from hist[cells][126][bins] ----
// (1) one thread per (cell, type): E = sum of bins in fp64 (bin order), learned
//     direction weights (R20 quantization, learned only) and their u32 prefix.
__global__ void k_dir_type_tables(const float *hist, int n_cells, int nb, double *E, uint32_t *dir_prefix) {
    int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n_cells * 126) return;
    const float *h = hist + (size_t)id * nb;
    double e = 0.0;
    float hmax = 0.0f;
    for (int b = 0; b < nb; b++) {
        float v = h[b];
        e += (double)v;
        hmax = fmaxf(hmax, v);
    }
    E[id] = e;
    uint32_t acc = 0;
    uint32_t *dp = dir_prefix + (size_t)id * nb;
    for (int b = 0; b < nb; b++) {
        uint32_t wb = 0;
        float v = h[b];
        if (v > 0.0f && hmax > 0.0f) {
            wb = (uint32_t)floorf(__fmul_rn(__fdiv_rn(v, hmax), 1048576.0f));
            if (wb < 1u) wb = 1u;
        }
        acc += wb;
        dp[b] = acc;
    }
}
// (2) one thread per cell: length mixture (Eqs. 10, 13) and per-length type tables (Eq. 11)
__global__ void k_dir_cell_tables(const double *E, int n_cells, uint64_t *n_prefix, uint64_t *type_prefix) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const double *e = E + (size_t)c * 126;
    const uint32_t P0[6] = {20, 20, 20, 20, 20, 19};
    double En[6], emax = 0.0;
    for (int n = 1; n <= 6; n++) {
        double s = 0.0;
        for (int m = 0; m < (1 << n); m++) s += e[(1 << n) - 2 + m];
        En[n - 1] = s;
        emax = fmax(emax, s);
    }
    uint64_t Wn[6], sumW = 0;
    for (int n = 0; n < 6; n++) {
        uint64_t w = 0;
        if (En[n] > 0.0 && emax > 0.0) {
            w = (uint64_t)floor(__dmul_rn(__ddiv_rn(En[n], emax), 1048576.0));
            if (w < 1u) w = 1u;
        }
        Wn[n] = w;
        sumW += w;
    }
    uint64_t acc = 0;
    for (int n = 0; n < 6; n++) {
        acc += sumW == 0 ? (uint64_t)P0[n] : (uint64_t)P0[n] * sumW + 119ull * Wn[n];
        n_prefix[(size_t)c * 6 + n] = acc;
    }
    for (int n = 1; n <= 6; n++) {
        int g0 = (1 << n) - 2, gn = 1 << n;
        double gmax = 0.0;
        for (int m = 0; m < gn; m++) gmax = fmax(gmax, e[g0 + m]);
        uint64_t a2 = 0;
        for (int m = 0; m < gn; m++) {
            uint64_t w = 0;
            if (e[g0 + m] > 0.0 && gmax > 0.0) {
                w = (uint64_t)floor(__dmul_rn(__ddiv_rn(e[g0 + m], gmax), 1048576.0));
                if (w < 1u) w = 1u;
            }
            a2 += w;
            type_prefix[(size_t)c * 126 + g0 + m] = a2;
        }
    }
}

static mpg_status build_dir_tables(mpg_guide *g, const float *hist, cudaStream_t st) {
    int nt = g->n_cells * 126;
    COUNT_LAUNCH(1);
    k_dir_type_tables<<<(nt + 127) / 128, 128, 0, st>>>(hist, g->n_cells, g->n_bins, g->type_energy, g->dir_prefix);
    CUDA_TRY(cudaPeekAtLastError());
    COUNT_LAUNCH(1);
    k_dir_cell_tables<<<(g->n_cells + 127) / 128, 128, 0, st>>>(g->type_energy, g->n_cells, g->n_prefix,
                                                                 g->type_prefix);
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}

// accumulate for the typed direction guide: hist[cell(x_D)][type(n,tau)][bin(w_D*)] += w (Eq. 9)
__global__ void k_accumulate_dir(const mpg_guide_desc g, const float4 *xD, int spp, int64_t n, const float4 *chain0,
                                 const uint8_t *status, const float *w, const uint16_t *ctype, float *hist) {
    const int nb = g.bins_x * g.bins_y;
    const int lane = threadIdx.x & 31;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = base + threadIdx.x;
        long long key = -1;
        float val = 0.f;
        if (i < n && status[i] == 0 && w[i] > 0.f) {
            uint32_t ct = ctype[i];
            int kk = (int)(ct & 15u);
            uint32_t tau = ct >> 4;
            float3 xd = xyz(xD[i / spp]);
            float3 x1 = xyz(chain0[i]);
            int cx = (int)floorf(FD(FM(FS(xd.x, g.grid_origin[0]), (float)g.cells_x), g.grid_extent[0]));
            int cz = (int)floorf(FD(FM(FS(xd.z, g.grid_origin[1]), (float)g.cells_y), g.grid_extent[1]));
            cx = min(max(cx, 0), g.cells_x - 1);
            cz = min(max(cz, 0), g.cells_y - 1);
            float dx = FS(x1.x, xd.x), dy = FS(x1.y, xd.y), dz = FS(x1.z, xd.z);
            float l = __fsqrt_rn(FA(FA(FM(dx, dx), FM(dy, dy)), FM(dz, dz)));
            float u = FD(dy, l);
            float v = FD(FA(atan2f(dz, dx), 3.14159265358979323846f), 6.28318530717958647692f);
            int bu = min(max((int)floorf(FM(u, (float)g.bins_x)), 0), g.bins_x - 1);
            int bv = min(max((int)floorf(FM(v, (float)g.bins_y)), 0), g.bins_y - 1);
            if (kk >= 1 && kk <= 6) {
                int type = (1 << kk) - 2 + (int)tau;
                key = ((long long)(cz * g.cells_x + cx) * 126 + type) * nb + bv * g.bins_x + bu;
                val = w[i];
            }
        }
        unsigned grp = __match_any_sync(MPG_FULL, key);
        float sum = 0.f;
        for (int j = 0; j < 32; j++) {
            float vj = __shfl_sync(MPG_FULL, val, j);
            if (grp & (1u << j)) sum += vj;
        }
        if (key >= 0 && lane == __ffs(grp) - 1) atomicAdd(hist + key, sum);
    }
}

extern "C" mpg_status mpg_guide_upload(mpg_guide *g, const float *energy, void *stream) {
    ARG_CHECK(g && energy, "NULL argument");
    ARG_CHECK(!g->stree, "STree guide: use mpg_guide_set_samples + mpg_guide_rebuild");
    if (g->desc.domain == 1) {
        mpg_status st = build_dir_tables(g, energy, as_stream(stream));
        if (st != MPG_OK) return st;
    } else {
        COUNT_LAUNCH(1);
        k_guide_tables<<<g->n_cells, GT_THREADS, 0, as_stream(stream)>>>(energy, g->n_bins, g->prefix);
    }
    CUDA_TRY(cudaPeekAtLastError());
    CUDA_TRY(cudaMemsetAsync(g->hist, 0, sizeof(float) * (size_t)g->n_cells * g->n_types * g->n_bins,
                             as_stream(stream)));
    g->ready = true;
    return MPG_OK;
}

static mpg_status stree_build(StreeState *T, cudaStream_t st);
static void stree_clear(StreeState *T);
extern "C" mpg_status mpg_guide_reset(mpg_guide *g, void *stream) {
    ARG_CHECK(g, "NULL guide");
    if (g->stree) {
        stree_clear(g->stree);
        return stree_build(g->stree, as_stream(stream));
    }
    CUDA_TRY(cudaMemsetAsync(g->hist, 0, sizeof(float) * (size_t)g->n_cells * g->n_types * g->n_bins,
                             as_stream(stream)));
    if (g->desc.domain == 1) {
        mpg_status st = build_dir_tables(g, g->hist, as_stream(stream));
        if (st != MPG_OK) return st;
    } else {
        COUNT_LAUNCH(1);
        k_guide_tables<<<g->n_cells, GT_THREADS, 0, as_stream(stream)>>>(g->hist, g->n_bins, g->prefix);
    }
    CUDA_TRY(cudaPeekAtLastError());
    g->ready = true;
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_accumulate(mpg_guide *g, const mpg_query *q, const mpg_walk_buf *wb, int64_t n,
                                           void *stream) {
    ARG_CHECK(g && !g->stree, "STree guide: use mpg_guide_record_samples");
    ARG_CHECK(g && q && wb && q->xD && wb->chain && wb->status && wb->w, "NULL argument");
    ARG_CHECK(q->spp >= 1 && n == q->n_recv * q->spp, "n must equal n_recv*spp");
    if (n == 0) return MPG_OK;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    if (g->desc.domain == 1) {
        ARG_CHECK(wb->ctype, "typed direction guide needs walk ctype");
        COUNT_LAUNCH(1);
        k_accumulate_dir<<<blocks, 256, 0, as_stream(stream)>>>(g->desc, (const float4 *)q->xD, q->spp, n,
                                                                (const float4 *)wb->chain, wb->status, wb->w,
                                                                wb->ctype, g->hist);
    } else {
        COUNT_LAUNCH(1);
        k_accumulate<<<blocks, 256, 0, as_stream(stream)>>>(g->desc, (const float4 *)q->xD, q->spp, n,
                                                            (const float4 *)wb->chain, wb->status, wb->w, g->hist);
    }
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_rebuild(mpg_guide *g, void *stream) {
    ARG_CHECK(g, "NULL guide");
    if (g->stree) return stree_build(g->stree, as_stream(stream));
    if (g->desc.domain == 1) {
        mpg_status st = build_dir_tables(g, g->hist, as_stream(stream));
        if (st != MPG_OK) return st;
    } else {
        COUNT_LAUNCH(1);
        k_guide_tables<<<g->n_cells, GT_THREADS, 0, as_stream(stream)>>>(g->hist, g->n_bins, g->prefix);
    }
    CUDA_TRY(cudaPeekAtLastError());
    CUDA_TRY(cudaMemsetAsync(g->hist, 0, sizeof(float) * (size_t)g->n_cells * g->n_types * g->n_bins,
                             as_stream(stream)));
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_download(const mpg_guide *g, float *energy, uint64_t *prefix, void *stream) {
    ARG_CHECK(g && !g->stree, "NULL guide or STree guide (use mpg_guide_download_stree)");
    size_t ne = (size_t)g->n_cells * g->n_types * g->n_bins;
    if (energy) CUDA_TRY(cudaMemcpyAsync(energy, g->hist, ne * sizeof(float), cudaMemcpyDeviceToDevice, as_stream(stream)));
    if (prefix) {
        ARG_CHECK(g->desc.domain == 0, "domain-1 tables: use mpg_guide_download_dir_tables");
        CUDA_TRY(cudaMemcpyAsync(prefix, g->prefix, ne * sizeof(uint64_t), cudaMemcpyDeviceToDevice, as_stream(stream)));
    }
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_set_histogram(mpg_guide *g, const float *energy, void *stream) {
    ARG_CHECK(g && energy, "NULL argument");
    ARG_CHECK(!g->stree, "STree guide: use mpg_guide_set_samples");
    size_t ne = (size_t)g->n_cells * g->n_types * g->n_bins;
    CUDA_TRY(cudaMemcpyAsync(g->hist, energy, ne * sizeof(float), cudaMemcpyDeviceToDevice, as_stream(stream)));
    return MPG_OK;
}

extern "C" mpg_status mpg_guide_download_dir_tables(const mpg_guide *g, uint64_t *n_prefix, uint64_t *type_prefix,
                                                    uint32_t *dir_prefix, void *stream) {
    ARG_CHECK(g && g->desc.domain == 1, "needs a typed direction guide");
    cudaStream_t s = as_stream(stream);
    if (n_prefix) CUDA_TRY(cudaMemcpyAsync(n_prefix, g->n_prefix, (size_t)g->n_cells * 6 * 8, cudaMemcpyDeviceToDevice, s));
    if (type_prefix)
        CUDA_TRY(cudaMemcpyAsync(type_prefix, g->type_prefix, (size_t)g->n_cells * 126 * 8, cudaMemcpyDeviceToDevice, s));
    if (dir_prefix)
        CUDA_TRY(cudaMemcpyAsync(dir_prefix, g->dir_prefix, (size_t)g->n_cells * 126 * g->n_bins * 4,
                                 cudaMemcpyDeviceToDevice, s));
    return MPG_OK;
}

#include "stree.cuh"
#include "photons.cuh"

// ----------------------------------------------------------------------------
// seeds
// ----------------------------------------------------------------------------
static mpg_status make_seed_ctx(const mpg_scene *scene, const mpg_guide *guide, const mpg_sampler_desc *sd,
                                const mpg_walk_opts *o, SeedCtx &g) {
    memset(&g, 0, sizeof(g));
    ARG_CHECK(sd->k >= 1 && sd->k <= MPG_KMAX, "k must be in [1, 8]");
    ARG_CHECK(sd->mode >= 0 && sd->mode <= 4, "bad sampler mode");
    if (sd->mode >= 3) ARG_CHECK(sd->k == 6, "GUIDE_DIR / GUIDE_STREE sample n <= 6: set k = 6");
    ARG_CHECK(sd->surf_id >= 0 && sd->surf_id < scene->d.n_surf, "sampler surf_id out of range");
    const DSurf &f = scene->d.surf[sd->surf_id];
    if (sd->mode == 0) ARG_CHECK(f.kind == 0, "CAP sampler needs a sphere");
    if (sd->mode == 1) ARG_CHECK(f.kind == 2, "TRIANGLE sampler needs a mesh");
    g.mode = sd->mode;
    g.surf_id = sd->surf_id;
    g.k = sd->k;
    g.tau = sd->tau & ((1u << sd->k) - 1u);
    g.seed = o->seed;
    if (sd->mode == 4) {
        ARG_CHECK(guide && guide->stree && guide->ready, "GUIDE_STREE sampler needs an STree guide");
        const StreeState *T = guide->stree;
        g.root_ref = T->root_ref;
        g.nodes = T->nodes.p;
        g.grp_off = T->grp_off.p;
        g.lobe_prefix = T->lobe_prefix.p;
        g.lobe_mu = T->lobe_mu.p;
        g.n_prefix = T->n_prefix.p;
        g.type_prefix = T->type_prefix.p;
        g.leaf_own = T->leaf_own.p;
        g.selective = (o->flags & MPG_FLAG_SELECTIVE) != 0;
        return MPG_OK;
    }
    if (sd->mode >= 2) {
        ARG_CHECK(guide && !guide->stree && guide->ready, "guided sampler needs an uploaded/reset guide");
        ARG_CHECK(guide->desc.domain == (sd->mode == 3 ? 1 : 0), "sampler mode / guide domain mismatch");
        const mpg_guide_desc &d = guide->desc;
        g.gox = d.grid_origin[0]; g.goz = d.grid_origin[1]; g.gex = d.grid_extent[0]; g.gez = d.grid_extent[1];
        g.cells_x = d.cells_x; g.cells_y = d.cells_y; g.bins_x = d.bins_x; g.bins_y = d.bins_y;
        g.uvox = d.uv_origin[0]; g.uvoz = d.uv_origin[1]; g.uvsx = d.uv_scale[0]; g.uvsz = d.uv_scale[1];
        g.uv_y = d.uv_plane_y;
        g.prefix = guide->prefix;
        g.n_prefix = guide->n_prefix;
        g.type_prefix = guide->type_prefix;
        g.dir_prefix = guide->dir_prefix;
    }
    return MPG_OK;
}

// The guided (u,v) sampler (mode 2) stages the prefix table of a cell in shared memory when all
// of a block's walks fall in that one cell (consecutive walks are consecutive receivers along a
// cell row: for configs[2] a 256-walk block spans 64 receivers of a 128-receiver-wide cell); the
// binary search then reads shared memory instead of L1/L2 (north_star).
__global__ void k_seeds(const DScene S, const SeedCtx g, const float4 *xD, int64_t n, int spp, uint64_t base,
                        float4 *xL, float4 *tgt, int *bin, uint32_t *ctype, float *pn, int stage_bins) {
    extern __shared__ unsigned long long s_pf[];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += stride) {   // block-uniform chunks
        const int64_t i = i0 + threadIdx.x;
        int stage_cell = -1;
        if (stage_bins) {
            const int c0 = seed_cell(g, xyz(xD[i0 / spp]));
            const int c = i < n ? seed_cell(g, xyz(xD[i / spp])) : c0;
            __syncthreads();                                   // previous chunk done with s_pf
            if (__syncthreads_and(c == c0)) {
                const unsigned long long *src = (const unsigned long long *)g.prefix + (size_t)c0 * stage_bins;
                for (int b = threadIdx.x; b < stage_bins; b += blockDim.x) s_pf[b] = __ldg(src + b);
                stage_cell = c0;
            }
            __syncthreads();
        }
        if (i >= n) continue;
        uint64_t wid = base + (uint64_t)i;
        float3 l;
        int lid;
        float pdf = sample_light(S, g.seed, wid, l, lid);
        xL[i] = make_float4(l.x, l.y, l.z, pdf);
        SeedRes sr;
        bool ok = seed_target(S, g, wid, 0u, xyz(xD[i / spp]), l, sr, stage_bins ? s_pf : nullptr, stage_cell);
        tgt[i] = make_float4(sr.tgt.x, sr.tgt.y, sr.tgt.z, 0.f);
        bin[i] = ok ? sr.bin : (sr.bin == -3 ? -3 : -2);   // -3: inactive (R36), -2: seed failed
        if (ctype) ctype[i] = (uint32_t)sr.n | ((sr.bits & 255u) << 4) | ((sr.learned ? 1u : 0u) << 12);
        if (pn) pn[i] = sr.Pn;
    }
}

static int g_num_sms = 0;
static int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

extern "C" mpg_status mpg_sample_seeds(const mpg_scene *scene, const mpg_guide *guide, const mpg_sampler_desc *sd,
                                       const mpg_query *q, const mpg_walk_opts *o, mpg_seed_buf *sb, void *stream) {
    ARG_CHECK(scene && sd && q && o && sb, "NULL argument");
    ARG_CHECK(q->n_recv >= 0 && q->spp >= 1, "bad query sizes");
    SeedCtx g;
    mpg_status st = make_seed_ctx(scene, guide, sd, o, g);
    if (st != MPG_OK) return st;
    int64_t n = q->n_recv * q->spp;
    if (n == 0) return MPG_OK;
    ARG_CHECK(q->xD && sb->xL && sb->target && sb->bin, "NULL query/seed array");
    int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    const int nb = g.bins_x * g.bins_y;
    // staging measured slower on configs[2] (k_seeds 0.72 vs 0.62 ms: a block loads the whole
    // 8 KB table for ~10 probes per walk that L1 serves anyway) -> opt-in (MPG_STAGE=1)
    static const bool want_stage = getenv("MPG_STAGE") && atoi(getenv("MPG_STAGE")) != 0;
    const int stage = (want_stage && g.mode == MPG_SEED_GUIDE_UV && nb > 0 && nb <= 6144) ? nb : 0;
    COUNT_LAUNCH(1);
    k_seeds<<<blocks, 256, (size_t)stage * 8, as_stream(stream)>>>(scene->d, g, (const float4 *)q->xD, n, q->spp,
                                                                   o->walk_id_base, (float4 *)sb->xL,
                                                                   (float4 *)sb->target, sb->bin, sb->ctype, sb->pn,
                                                                   stage);
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}

// ----------------------------------------------------------------------------
// walk
// ----------------------------------------------------------------------------
#ifdef MPG_TIMELINE
// diagnostic build only: copy out (and zero) the k_walk activity timeline
extern "C" int mpg_debug_timeline(unsigned long long *host4096, unsigned shift, unsigned long long *host256) {
    cudaDeviceSynchronize();
    cudaMemcpyToSymbol(g_tl_shift, &shift, sizeof(shift));
    cudaMemcpyFromSymbol(host4096, g_tl, sizeof(g_tl));
    cudaMemcpyFromSymbol(host256, g_nh, sizeof(g_nh));
    static unsigned long long zero[1024 * 4];
    cudaMemcpyToSymbol(g_tl, zero, sizeof(g_tl));
    cudaMemcpyToSymbol(g_nh, zero, sizeof(g_nh));
    return 0;
}
#endif
static float *g_dbg = nullptr;
static int64_t g_dbg_n = 0;
static int g_dbg_stride = 0;
extern "C" mpg_status mpg_debug_trace(float *buf, int64_t n_walks, int32_t stride) {
    g_dbg = buf;
    g_dbg_n = buf ? n_walks : 0;
    g_dbg_stride = stride;
    return MPG_OK;
}

// persistent-kernel workspace: trial header, hard entries
// (walks unresolved after LOCAL_TRIALS sequential trials), item ring
// Sequential trials run in the lane before a walk becomes a hard entry.  Measured
// (ms/step, configs 1/2/3/4): 1 -> 66/508/337/391, 2 -> 62/497/337/386,
// 4 -> 61.5/474/335/377, 8 -> 62.6/451/335/377: with many walks per launch the
// primaries keep every lane busy and in-lane trials are cheaper than items, with
// few the parallel items shorten the tail.  Re-measured in round 2 with the batched attempt
// boundaries (configs[2], 16.8 M walks): 2 -> 292, 4 -> 268, 8 -> 243, 16 -> 229, 32 -> 225,
// 64..1024 -> 225 ms; configs[1] (1 M walks) flat from 4 to 1024; configs[3]/[4] flat or +1 %.
#ifdef MPG_LOCAL_TRIALS
#define LOCAL_TRIALS(n) ((uint32_t)MPG_LOCAL_TRIALS)
#else
#define LOCAL_TRIALS(n) ((n) >= (int64_t)4 << 20 ? 32u : 4u)
#endif
struct MKLayout {
    uint32_t H, C;
    size_t th, e_walk, e_psurf, e_pct, e_best, e_pending, e_issued, e_batch, items, skey, skey2, sval, sval2, stemp,
        stemp_bytes, total;
};
static MKLayout mk_layout(int64_t n) {
    MKLayout L;
    int64_t nn = std::max<int64_t>(n, 1);
    L.H = (uint32_t)std::min<int64_t>(nn, 1 << 22);
    L.C = 8u * L.H + 65536u;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 255) & ~(size_t)255; return r; };
    L.th = take(sizeof(TrialHdr));
    L.e_walk = take(8ull * L.H);
    L.e_psurf = take(4ull * L.H); L.e_pct = take(4ull * L.H); L.e_best = take(4ull * L.H);
    L.e_pending = take(4ull * L.H); L.e_issued = take(4ull * L.H); L.e_batch = take(4ull * L.H);
    L.items = take(8ull * L.C);
    // MPG_FLAG_SORT: keys / permutation (double-buffered) and radix-sort scratch
    L.skey = take(4ull * nn); L.skey2 = take(4ull * nn); L.sval = take(4ull * nn); L.sval2 = take(4ull * nn);
    L.stemp_bytes = 16ull * nn + (8u << 20);
    L.stemp = take(L.stemp_bytes);
    L.total = o;
    return L;
}

// MPG_FLAG_SORT keys: receiver cell (4 bits per axis, cells of extent/16, Morton)
// above the seed direction (octahedral map, 9 bits per axis, Morton); with a
// per-sample chain length (configs[4], ctype != NULL) the length goes on top
// (equal k walk together: the rolled per-vertex loops run the warp's max k) and
// the direction keeps 8 bits per axis.  Walks without a seed last.  Values: walk
// indices.
__device__ __forceinline__ uint32_t mpg_spread2(uint32_t v) { // 9 bits -> every 2nd bit
    v &= 0x1ffu;
    v = (v | (v << 8)) & 0x00ff00ffu;
    v = (v | (v << 4)) & 0x0f0f0f0fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__global__ void k_sort_keys(const float4 *xD, const float4 *tgt, const int *bin, const uint32_t *ctype, int64_t n,
                            int spp, float cell, uint32_t *key, uint32_t *val) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x) {
        val[w] = (uint32_t)w;
        if (bin[w] == -2) { key[w] = 0xffffffffu; continue; }
        float3 p = xyz(xD[w / spp]);
        float3 d = xyz(tgt[w]) - p;
        float l1 = fabsf(d.x) + fabsf(d.y) + fabsf(d.z);
        float u = l1 > 0.f ? d.x / l1 : 0.f, v = l1 > 0.f ? d.z / l1 : 0.f;
        if (d.y < 0.f) { // fold the lower hemisphere
            float uu = (1.f - fabsf(v)) * copysignf(1.f, u), vv = (1.f - fabsf(u)) * copysignf(1.f, v);
            u = uu; v = vv;
        }
        uint32_t qu = (uint32_t)min(511.f, fmaxf(0.f, (u * 0.5f + 0.5f) * 512.f));
        uint32_t qv = (uint32_t)min(511.f, fmaxf(0.f, (v * 0.5f + 0.5f) * 512.f));
        uint32_t dir = mpg_spread2(qu) | (mpg_spread2(qv) << 1);             // 18 bits
        uint32_t cx = (uint32_t)floorf(p.x / cell) & 15u, cy = (uint32_t)floorf(p.y / cell) & 15u,
                 cz = (uint32_t)floorf(p.z / cell) & 15u;
        uint32_t pos = 0;
        for (int b = 0; b < 4; b++)
            pos |= (((cx >> b) & 1u) << (3 * b)) | (((cy >> b) & 1u) << (3 * b + 1)) | (((cz >> b) & 1u) << (3 * b + 2));
        if (ctype) {   // per-sample chain length (configs[4]): group equal lengths first
            const uint32_t len = min(__ldg(ctype + w) & 15u, 7u);
            key[w] = (len << 28) | (pos << 16) | (dir >> 2);                     // 31 bits
        } else {
            key[w] = (pos << 18) | dir;                                          // 30 bits
        }
    }
}
static size_t mk_ws_bytes(int64_t n) { return mk_layout(n).total; }
// recip_repeats scratch after the walk workspace: w_r [n] f32, trials_r [n] u32, stats
static size_t rep_bytes(int64_t n) { return ((size_t)n * 12 + sizeof(mpg_walk_stats) + 767) & ~(size_t)255; }

static size_t rep_offset(int64_t n, int k) {
    (void)k;
    return (mk_ws_bytes(n) + 255) & ~(size_t)255;
}
// R x M: w += w_r, trials += trials_r (then w *= scale on the last repetition); work
// counters of the repetition added to the caller's stats (walks/converged count one pass)
__global__ void k_repeat_accum(float *w, uint32_t *trials, const float *w_r, const uint32_t *t_r, int64_t n,
                               unsigned long long *stats, const unsigned long long *s_r, float scale) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        w[i] = __fmul_rn(__fadd_rn(w[i], w_r[i]), scale);
        trials[i] += t_r[i];
    }
    if (stats && blockIdx.x == 0 && threadIdx.x < 11) {
        // mpg_walk_stats: walks, converged, newton_iters, primary_iters, attempts, rays, trials, truncated,
        // node_visits, tri_tests, vertex_iters
        const int f = threadIdx.x;
        if (f != 0 && f != 1 && f != 3) atomicAdd(stats + f, s_r[f]);
    }
}

static mpg_status walk_dispatch(const mpg_scene *scene, const SeedCtx &g, const mpg_sampler_desc *sd,
                                const mpg_walk_opts *o, const WalkParams &P, void *workspace, size_t workspace_bytes,
                                cudaStream_t s);

extern "C" size_t mpg_walk_workspace_size(int64_t n, const mpg_sampler_desc *sampler, const mpg_walk_opts *opts) {
    int k = sampler ? std::max(1, std::min(MPG_KMAX, (int)sampler->k)) : MPG_KMAX;
    (void)opts; // one size serves both paths (+ the per-repetition buffers of recip_repeats)
    return rep_offset(n, k) + rep_bytes(n);
}

// persisting-L2 carve-out for the traversal data (MPG_L2_PERSIST_MB, default below; 0 = off)
#ifndef MPG_L2_PERSIST_DEFAULT_MB
#define MPG_L2_PERSIST_DEFAULT_MB 0
#endif
static size_t l2_max_window() {
    static size_t v = 0;
    if (!v) {
        int dev = 0, w = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&w, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        v = w > 0 ? (size_t)w : 1;
    }
    return v;
}
static size_t l2_persist_bytes() {
    static long long v = -1;
    if (v < 0) {
        const char *e = getenv("MPG_L2_PERSIST_MB");
        long long mb = e ? atoll(e) : MPG_L2_PERSIST_DEFAULT_MB;
        int dev = 0, mx = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
        v = std::min<long long>(mb << 20, mx);
        if (v > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)v) != cudaSuccess) v = 0;
        if (v < 0) v = 0;
    }
    return (size_t)v;
}

template <int KMAX, typename R, int MINB = (KMAX <= 2 ? MPG_WALK_MINB2 : MPG_WALK_MINB_LONG), bool GL = false,
          bool CMP = false>
static mpg_status launch_walk(const DScene &S, const SeedCtx &g, WalkParams P, cudaStream_t st, void *ws,
                              bool sort) {
    const bool wide = S.bvh_w == 4;
    static int occ2 = 0, occ4 = 0;
    int &occ = wide ? occ4 : occ2;
    if (!occ) {
        // shared-memory carve-out preference (MPG_CARVEOUT percent, unset: driver default);
        // the kernel needs 1.7 KB of shared memory per block, the rest of the unified
        // L1/shared array can cache nodes and the lanes' local memory
        if (const char *e = getenv("MPG_CARVEOUT")) {
            int pc = atoi(e);
            CUDA_TRY(cudaFuncSetAttribute(k_walk<KMAX, R, 4, MINB, GL, CMP>, cudaFuncAttributePreferredSharedMemoryCarveout, pc));
            CUDA_TRY(cudaFuncSetAttribute(k_walk<KMAX, R, 2, MINB, GL, CMP>, cudaFuncAttributePreferredSharedMemoryCarveout, pc));
        }
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &occ, wide ? k_walk<KMAX, R, 4, MINB, GL, CMP> : k_walk<KMAX, R, 2, MINB, GL, CMP>, 128, 0));
        if (occ <= 0) occ = 1;
    }
    MKLayout L = mk_layout(P.n);
    char *b = (char *)ws;
    P.local_trials = LOCAL_TRIALS(P.n);
    P.item_b0 = 4u;
    P.item_grow = 1u;
    P.backoff_max = 32768u;
    if (const char *v = getenv("MPG_LOCAL_TRIALS")) P.local_trials = (uint32_t)atoi(v);
    if (const char *v = getenv("MPG_ITEM_B0")) P.item_b0 = std::max(1, atoi(v));
    if (const char *v = getenv("MPG_ITEM_GROW")) P.item_grow = std::max(1, std::min(4, atoi(v)));
    P.item_grow_idle = 3u;   // x8 (measured x2/x4/x8: configs[1] 49.1/47.2/46.6 ms, [4] 13.2/12.5/11.8, [2,3] flat)
    P.idle_backlog = 0u;   // set from the grid below
    P.item_b0_idle = 4u;
    if (const char *v = getenv("MPG_ITEM_B0_IDLE")) P.item_b0_idle = std::max(1, atoi(v));
    if (const char *v = getenv("MPG_ITEM_GROW_IDLE")) P.item_grow_idle = std::max(1, std::min(4, atoi(v)));
    if (const char *v = getenv("MPG_BACKOFF_MAX")) P.backoff_max = std::max(32, atoi(v));
    // attempt boundaries (end / fetch / seed sections) served in batches (kernels for k <= 2 and the
    // mixed-length kernel).  Measured, ms per step at svc_min / svc_wait = 1/1 (every pass, as before),
    // 2/2, 4/3, 8/4, 8/8, 12/12, 16/12, 24/16: configs[2] 292.4 / 281.1 / 266.5 / 258.4 / 249.2 /
    // 242.8 / 243.2 / 290.6; configs[1] 43.9 / 43.9 / 43.1 / 42.6 / 42.5 / 42.6; configs[4] 217.9 -> 213.9
    // at 12/12; fixed k = 6 (configs[3]) 156.4 -> 158-160: not used there
    P.svc_min = 12u;
    P.svc_wait = 12u;
    if (const char *v = getenv("MPG_SVC_MIN")) P.svc_min = (uint32_t)std::max(1, std::min(32, atoi(v)));
    if (const char *v = getenv("MPG_SVC_WAIT")) P.svc_wait = (uint32_t)std::max(1, atoi(v));
    P.hard_cap = L.H;
    // tickets index the ring only below item_cap: it bounds both the reads and the clear;
    // a full ring (or entry table) makes the walk continue its trials sequentially
    P.item_cap = P.trials_on ? L.C : 0u;
    // test knobs: shrink the entry table / item ring to exercise the sequential fallbacks
    if (const char *v = getenv("MPG_TEST_HARD_CAP")) P.hard_cap = std::min<uint32_t>(P.hard_cap, (uint32_t)atoi(v));
    if (const char *v = getenv("MPG_TEST_ITEM_CAP")) P.item_cap = std::min<uint32_t>(P.item_cap, (uint32_t)atoi(v));
    P.th = (TrialHdr *)(b + L.th);
    P.e_walk = (int64_t *)(b + L.e_walk);
    P.e_psurf = (uint32_t *)(b + L.e_psurf); P.e_pct = (uint32_t *)(b + L.e_pct); P.e_best = (uint32_t *)(b + L.e_best);
    P.e_pending = (uint32_t *)(b + L.e_pending); P.e_issued = (uint32_t *)(b + L.e_issued);
    P.e_batch = (uint32_t *)(b + L.e_batch);
    P.items = (unsigned long long *)(b + L.items);
    CUDA_TRY(cudaMemsetAsync(P.th, 0, sizeof(TrialHdr), st));
    if (P.trials_on) CUDA_TRY(cudaMemsetAsync(P.items, 0xff, 8ull * P.item_cap, st));
    P.perm = nullptr;
    if (sort && P.n > 1) {
        uint32_t *k0 = (uint32_t *)(b + L.skey), *k1 = (uint32_t *)(b + L.skey2);
        uint32_t *v0 = (uint32_t *)(b + L.sval), *v1 = (uint32_t *)(b + L.sval2);
        int gk = (int)std::min<int64_t>((P.n + 255) / 256, (int64_t)num_sms() * 8);
        COUNT_LAUNCH(1);
        const uint32_t *len = g.mode == MPG_SEED_GUIDE_DIR ? P.seed_ctype : nullptr;   // per-sample n
        k_sort_keys<<<gk, 256, 0, st>>>(P.xD, P.seed_tgt, P.seed_bin, len, P.n, P.spp, S.extent / 16.0f, k0, v0);
        CUDA_TRY(cudaPeekAtLastError());
        size_t tb = 0;
        const int kbits = len ? 31 : 30;
        CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, (int)P.n, 0, kbits, st));
        if (tb > L.stemp_bytes) return fail(MPG_ERR_INVALID_ARG, "sort scratch larger than reserved");
        COUNT_LAUNCH(4);   // cub onesweep: histogram + 3 passes of 10 bits (library launches, counted)
        CUDA_TRY(cub::DeviceRadixSort::SortPairs(b + L.stemp, tb, k0, k1, v0, v1, (int)P.n, 0, kbits, st));
        P.perm = v1;
    }
    int64_t want = (P.n + 127) / 128;
    int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * occ);
    {
        int div = 8;   // idle: fewer unclaimed items than 1/div of the lanes
        if (const char *v = getenv("MPG_IDLE_DIV")) div = std::max(0, atoi(v));
        P.idle_backlog = div ? (uint32_t)(blocks * 128 / div) : 0x7fffffffu;   // 0: any backlog
    }
    COUNT_LAUNCH(1);
    // L2 access-policy window over the traversal data (nodes + triangle positions,
    // contiguous): persisting, so the walk's local-memory traffic (per-lane chain state
    // and traversal stacks) cannot evict the BVH from L2 (configs[2]/[3] measured
    // ~1.7 TB/s DRAM at 55 % L2 hits without it).  MPG_L2_PERSIST_MB (0 = off).
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = 0;
    const size_t lim = l2_persist_bytes();
    if (lim && P.trav_bytes) {
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = (void *)S.nodes;
        attr[0].val.accessPolicyWindow.num_bytes = std::min(P.trav_bytes, l2_max_window());
        attr[0].val.accessPolicyWindow.hitRatio =
            std::min(1.0f, (float)lim / (float)attr[0].val.accessPolicyWindow.num_bytes);
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs = 1;
    }
    if (wide) CUDA_TRY(cudaLaunchKernelEx(&cfg, k_walk<KMAX, R, 4, MINB, GL, CMP>, S, g, P));
    else CUDA_TRY(cudaLaunchKernelEx(&cfg, k_walk<KMAX, R, 2, MINB, GL, CMP>, S, g, P));
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}

extern "C" mpg_status mpg_manifold_walk(const mpg_scene *scene, const mpg_guide *guide, const mpg_sampler_desc *sd,
                                        const mpg_query *q, const mpg_seed_buf *sb, const mpg_walk_opts *o,
                                        mpg_walk_buf *out, mpg_walk_stats *stats, void *workspace,
                                        size_t workspace_bytes, void *stream) {
    ARG_CHECK(scene && sd && q && sb && o && out, "NULL argument");
    ARG_CHECK(q->n_recv >= 0 && q->spp >= 1, "bad query sizes");
    if (q->n_recv > 0) {
        ARG_CHECK(q->xD && q->nD && sb->xL && sb->target && sb->bin, "NULL query/seed array");
        ARG_CHECK(out->chain && out->status && out->iters && out->G && out->T && out->w && out->trials,
                  "NULL output array");
    }
    ARG_CHECK(workspace && workspace_bytes >= mpg_walk_workspace_size(q->n_recv * q->spp, sd, o), "workspace too small");
    ARG_CHECK(q->n_recv * (int64_t)q->spp < (int64_t)1 << 31, "at most 2^31-1 walks per call");
    ARG_CHECK(o->max_iters >= 0 && o->max_iters < 65536 && o->tol > 0.f && o->beta0 > 0.f, "bad walk options");
    ARG_CHECK(!o->trials || o->k_max >= 1, "k_max must be >= 1");
    ARG_CHECK((o->flags & ~(MPG_FLAG_NEWTON_F64 | MPG_FLAG_SORT | MPG_FLAG_SELECTIVE)) == 0, "unknown walk flag");
    SeedCtx g;
    mpg_status st = make_seed_ctx(scene, guide, sd, o, g);
    if (st != MPG_OK) return st;
    WalkParams P;
    memset(&P, 0, sizeof(P));
    P.n_recv = q->n_recv;
    P.spp = q->spp;
    P.n = q->n_recv * q->spp;
    cudaStream_t s = as_stream(stream);
    if (stats) CUDA_TRY(cudaMemsetAsync(stats, 0, sizeof(mpg_walk_stats), s));
    if (P.n == 0) return MPG_OK;
    P.xD = (const float4 *)q->xD;
    P.nD = (const float4 *)q->nD;
    P.seed_xL = (const float4 *)sb->xL;
    P.seed_tgt = (const float4 *)sb->target;
    P.seed_bin = sb->bin;
    P.seed_ctype = sb->ctype;
    P.seed_pn = sb->pn;
    P.out_ctype = out->ctype;
    P.max_iters_long = o->max_iters_long;
    P.chain = (float4 *)out->chain;
    P.status = out->status;
    P.iters = out->iters;
    P.G = out->G; P.T = out->T; P.w = out->w;
    P.trials = out->trials;
    P.stats = (unsigned long long *)stats;
    P.max_iters = o->max_iters;
    P.trials_on = o->trials;
    P.k_max = o->k_max;
    P.tol = o->tol;
    P.beta0 = o->beta0;
    P.same_eps = o->same_chain_eps > 0.f ? o->same_chain_eps : 1e-4f * scene->d.extent;
    P.ray_eps = o->ray_eps > 0.f ? o->ray_eps : 1e-4f * scene->d.extent;
    P.walk_id_base = o->walk_id_base;
    P.trav_bytes = scene->trav_bytes;
    P.dbg = g_dbg;
    P.n_dbg = g_dbg_n;
    P.dbg_stride = g_dbg_stride;
    int k = g.k;
    if (sd->mode >= MPG_SEED_GUIDE_DIR)
        ARG_CHECK(sb->ctype && sb->pn && out->ctype, "GUIDE_DIR/STREE need seed ctype/pn and walk ctype arrays");
    const int M = std::max(1, (int)o->recip_repeats);
    ARG_CHECK(M == 1 || (o->trials && o->k_max < (1u << 20) && M <= 4096), "recip_repeats needs trials, k_max < 2^20, M <= 4096");
    if (M == 1) return walk_dispatch(scene, g, sd, o, P, workspace, workspace_bytes, s);
    // R x M: M independent trial sequences, averaged
    char *rb = (char *)workspace + rep_offset(P.n, k);
    float *w_r = (float *)rb;
    uint32_t *t_r = (uint32_t *)(rb + (size_t)P.n * 4);
    mpg_walk_stats *s_r = (mpg_walk_stats *)(((uintptr_t)(rb + (size_t)P.n * 8) + 255) & ~(uintptr_t)255);
    uint32_t *ps_r = (uint32_t *)(((uintptr_t)(s_r + 1) + 255) & ~(uintptr_t)255);
    WalkParams P0 = P;
    P0.psurf_out = ps_r;
    st = walk_dispatch(scene, g, sd, o, P0, workspace, workspace_bytes, s);
    if (st != MPG_OK) return st;
    for (int r = 1; r < M; r++) {
        WalkParams Pr = P;
        Pr.trial_base = (uint32_t)r << 20;
        Pr.w = w_r;
        Pr.trials = t_r;
        Pr.stats = (unsigned long long *)s_r;
        Pr.psurf_out = ps_r;
        Pr.trials_only = 1;
        CUDA_TRY(cudaMemsetAsync(s_r, 0, sizeof(mpg_walk_stats), s));
        st = walk_dispatch(scene, g, sd, o, Pr, workspace, workspace_bytes, s);
        if (st != MPG_OK) return st;
        COUNT_LAUNCH(1);
        k_repeat_accum<<<(int)std::min<int64_t>((P.n + 255) / 256, (int64_t)num_sms() * 8), 256, 0, s>>>(
            out->w, out->trials, w_r, t_r, P.n, (unsigned long long *)stats, (const unsigned long long *)s_r,
            r == M - 1 ? 1.0f / (float)M : 1.0f);
        CUDA_TRY(cudaPeekAtLastError());
    }
    return MPG_OK;
}

static mpg_status walk_dispatch(const mpg_scene *scene, const SeedCtx &g, const mpg_sampler_desc *sd,
                                const mpg_walk_opts *o, const WalkParams &P, void *workspace, size_t workspace_bytes,
                                cudaStream_t s) {
    const int k = g.k;
    const bool sort = (o->flags & MPG_FLAG_SORT) != 0, f64 = (o->flags & MPG_FLAG_NEWTON_F64) != 0;
    if (scene->glossy) {   // glossy chains (R37): kernels with the offset-normal code, k <= 6
        if (k > 6) return fail(MPG_ERR_UNSUPPORTED, "glossy chains support k <= 6");
        if (f64) {
            if (k <= 2) return launch_walk<2, double, MPG_WALK_MINB2, true>(scene->d, g, P, s, workspace, sort);
            return launch_walk<6, double, MPG_WALK_MINB_LONG, true>(scene->d, g, P, s, workspace, sort);
        }
        if (k <= 2) return launch_walk<2, float, MPG_WALK_MINB2, true>(scene->d, g, P, s, workspace, sort);
        return launch_walk<6, float, MPG_WALK_MINB_LONG, true>(scene->d, g, P, s, workspace, sort);
    }
#ifndef MPG_CMP_SHORT
#define MPG_CMP_SHORT 0   // compacted rounds for fixed k <= 2 (A/B knob; measured slower)
#endif
#ifndef MPG_CMP_LONG
#define MPG_CMP_LONG 0    // compacted rounds for fixed k in 3..6 (A/B knob)
#endif
    if (f64) {
        if (k <= 1) return launch_walk<1, double, MPG_WALK_MINB2, false, MPG_CMP_SHORT != 0>(scene->d, g, P, s, workspace, sort);
        if (k <= 2) return launch_walk<2, double, MPG_WALK_MINB2, false, MPG_CMP_SHORT != 0>(scene->d, g, P, s, workspace, sort);
        if (k <= 4) return launch_walk<4, double>(scene->d, g, P, s, workspace, sort);
        if (k <= 6) {
            // mixed chain lengths (configs[4]): see MPG_WALK_MINB_MIXED; compacted trace rounds
            // (MPG_COMPACT) measured faster there only
            if (sd->mode >= MPG_SEED_GUIDE_DIR)
                return launch_walk<6, double, MPG_WALK_MINB_MIXED, false, MPG_COMPACT != 0>(scene->d, g, P, s,
                                                                                          workspace, sort);
            return launch_walk<6, double, MPG_WALK_MINB_LONG, false, MPG_CMP_LONG != 0>(scene->d, g, P, s, workspace,
                                                                                        sort);
        }
        return launch_walk<8, double>(scene->d, g, P, s, workspace, sort);
    }
    if (k <= 1) return launch_walk<1, float>(scene->d, g, P, s, workspace, sort);
    if (k <= 2) return launch_walk<2, float>(scene->d, g, P, s, workspace, sort);
    if (k <= 4) return launch_walk<4, float>(scene->d, g, P, s, workspace, sort);
    if (k <= 6) return launch_walk<6, float>(scene->d, g, P, s, workspace, sort);
    return launch_walk<8, float>(scene->d, g, P, s, workspace, sort);
}

// ----------------------------------------------------------------------------
// estimator (Eq. 3)
// ----------------------------------------------------------------------------
__global__ void k_estimate(const float *w, int64_t n_recv, int spp, float *mean, float *var) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_recv; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0, s2 = 0.0;
        for (int j = 0; j < spp; j++) {
            double v = w[r * spp + j];
            s += v;
            s2 += v * v;
        }
        mean[r] = (float)(s / spp);
        if (var) var[r] = spp > 1 ? (float)((s2 - s * s / spp) / (spp - 1)) : 0.0f;
    }
}

extern "C" mpg_status mpg_estimate(const float *w, int64_t n_recv, int32_t spp, float *mean, float *var, void *stream) {
    ARG_CHECK(w && mean && n_recv >= 0 && spp >= 1, "bad argument");
    if (n_recv == 0) return MPG_OK;
    int blocks = (int)std::min<int64_t>((n_recv + 255) / 256, (int64_t)num_sms() * 8);
    COUNT_LAUNCH(1);
    k_estimate<<<blocks, 256, 0, as_stream(stream)>>>(w, n_recv, spp, mean, var);
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}

// splat (Eq. 3 over render passes): sum[r] += sum_j w[r*spp+j], sumsq[r] += (that pass mean)^2, fp64
__global__ void k_splat(const float *w, int64_t n_recv, int spp, double *sum, double *sumsq) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_recv; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < spp; j++) s += (double)w[r * spp + j];
        s /= spp;
        sum[r] += s;
        if (sumsq) sumsq[r] += s * s;
    }
}

extern "C" mpg_status mpg_splat(const float *w, int64_t n_recv, int32_t spp, double *sum, double *sumsq, void *stream) {
    ARG_CHECK(w && sum && n_recv >= 0 && spp >= 1, "bad argument");
    if (n_recv == 0) return MPG_OK;
    int blocks = (int)std::min<int64_t>((n_recv + 255) / 256, (int64_t)num_sms() * 8);
    COUNT_LAUNCH(1);
    k_splat<<<blocks, 256, 0, as_stream(stream)>>>(w, n_recv, spp, sum, sumsq);
    CUDA_TRY(cudaPeekAtLastError());
    return MPG_OK;
}

extern "C" const char *mpg_last_error(void) { return g_err.c_str(); }
extern "C" int32_t mpg_version(void) { return 1; }
extern "C" uint64_t mpg_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

// ----------------------------------------------------------------------------
// measurement helper (not on the walk path): the FP32 FFMA roof of this GPU,
// the denominator of bench.py's roofline ("measure with an FFMA
// microbenchmark on the box").  Every thread runs 8 independent FFMA chains
// (latency 4 cycles, so 2 warps per SM sub-partition already saturate the
// pipe); grid = SMs x 4 blocks of 256; best of `reps` launches.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ffma_peak(float *out, int iters, float b, float c) {
    float a0 = threadIdx.x * 1e-7f, a1 = a0 + 1.0f, a2 = a0 + 2.0f, a3 = a0 + 3.0f, a4 = a0 + 4.0f, a5 = a0 + 5.0f,
          a6 = a0 + 6.0f, a7 = a0 + 7.0f;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) {
            a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
            a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
        }
    }
    const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678f) out[0] = s;   // keeps the chains live
}

extern "C" mpg_status mpg_measure_fp32_peak(int32_t iters, int32_t reps, double *tflops, void *stream) {
    ARG_CHECK(tflops && iters > 0 && reps > 0, "bad argument");
    cudaStream_t s = as_stream(stream);
    float *d = nullptr;
    CUDA_TRY(cudaMallocAsync(&d, 4, s));
    const int blocks = num_sms() * 4;
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    double best = 0.0;
    for (int r = 0; r <= reps; r++) {   // r = 0: warm-up
        CUDA_TRY(cudaEventRecord(e0, s));
        COUNT_LAUNCH(1);
        k_ffma_peak<<<blocks, 256, 0, s>>>(d, iters, 0.999999f, 1e-6f);
        CUDA_TRY(cudaEventRecord(e1, s));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        const double flops = (double)blocks * 256.0 * iters * 16.0 * 8.0 * 2.0;
        if (r > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CUDA_TRY(cudaFreeAsync(d, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *tflops = best;
    return MPG_OK;
}

// ----------------------------------------------------------------------------
// online training schedule (reading R34): host logic of the
// progressive train/render loop, in passes of one walk per receiver
// ----------------------------------------------------------------------------
extern "C" mpg_status mpg_training_schedule(int64_t budget_passes, double train_frac, int64_t *iters,
                                            int32_t max_iters, int32_t *n_iters, int64_t *render_passes) {
    ARG_CHECK(budget_passes >= 0 && train_frac >= 0.0 && train_frac <= 1.0, "bad budget / training fraction");
    ARG_CHECK(n_iters && render_passes && (iters || max_iters == 0) && max_iters >= 0, "NULL argument");
    // "We stop the training stage immediately when 30% of the budget is already used"
    const int64_t T = (int64_t)std::floor(train_frac * (double)budget_passes);
    int32_t m = 0;
    int64_t used = 0, size = 1;   // "we double the sample count in each iteration"
    while (used < T) {
        ARG_CHECK(m < max_iters, "iters array too short");
        int64_t n = std::min(size, T - used);
        iters[m++] = n;
        used += n;
        if (used >= T) break;
        // "when a training iteration is finished, we start a new round if less than half of
        // the training budget is used.  Otherwise, we continue the current iteration until the
        // rendering stage starts"
        if (2 * used < T) size *= 2;
        else { iters[m - 1] += T - used; used = T; }
    }
    *n_iters = m;
    *render_passes = budget_passes - T;
    return MPG_OK;
}
