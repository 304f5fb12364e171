"""ctypes front end of the C oracle (oracle/mpg_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module.  It shares nothing with the CUDA library: it builds its own
shared object from oracle/mpg_oracle.c with gcc and marshals the seeded input
arrays of paper_2311_12818_b200/workloads.py (inputs only, no method
arithmetic) into the oracle's own records.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mpg_oracle.c")
LIB = os.path.join(HERE, "libmpg_oracle.so")
KMAX = 8

STATUS = {0: "CONVERGED", 1: "MAXITER", 2: "SEED_FAIL", 3: "BAD_SIDE", 4: "DEGENERATE", 5: "OCCLUDED", 6: "INACTIVE"}


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2, no FP contraction, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", LIB, SRC, "-lm"])
    return LIB


class Surface(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mat", C.c_int32), ("tri_begin", C.c_int32), ("tri_count", C.c_int32),
                ("eta_in", C.c_float), ("eta_out", C.c_float), ("reflectance", C.c_float), ("radius", C.c_float),
                ("center", C.c_float * 3), ("origin", C.c_float * 3), ("edge_u", C.c_float * 3),
                ("edge_v", C.c_float * 3), ("roughness", C.c_float)]


class Light(C.Structure):
    _fields_ = [("kind", C.c_int32), ("emit", C.c_float), ("position", C.c_float * 3), ("edge_u", C.c_float * 3),
                ("edge_v", C.c_float * 3)]


class SeedCfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("surf_id", C.c_int32), ("k", C.c_int32), ("tau", C.c_uint32),
                ("grid_origin", C.c_float * 2), ("grid_extent", C.c_float * 2), ("cells_x", C.c_int32),
                ("cells_y", C.c_int32), ("bins_x", C.c_int32), ("bins_y", C.c_int32), ("uv_origin", C.c_float * 2),
                ("uv_scale", C.c_float * 2), ("uv_plane_y", C.c_float), ("prefix", C.POINTER(C.c_uint64)),
                ("n_prefix", C.c_void_p), ("type_prefix", C.c_void_p), ("dir_prefix", C.c_void_p),
                ("root_ref", C.c_int32), ("pad_", C.c_int32), ("nodes", C.c_void_p), ("grp_off", C.c_void_p),
                ("lobe_prefix", C.c_void_p), ("lobe_mu", C.c_void_p), ("leaf_own", C.c_void_p)]


# STree + vMF guide: 48-byte sample record and tree node, as in mpg_oracle.c
GSAMPLE = np.dtype([("xD", np.float32, (3,)), ("xL", np.float32, (3,)), ("omega", np.float32, (3,)),
                    ("w", np.float32), ("type", np.int32), ("pad", np.int32)])
class PhotonDesc(C.Structure):
    _fields_ = [("n_photons", C.c_int64), ("seed", C.c_uint64), ("photon_id_base", C.c_uint64),
                ("plane_point", C.c_float * 3), ("plane_normal", C.c_float * 3), ("max_vertices", C.c_int32),
                ("ray_eps", C.c_float)]


SNODE = np.dtype([("split", np.float32), ("axis", np.int32), ("child", np.int32, (2,))])


class Opts(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("trials", C.c_int32), ("k_max", C.c_uint32), ("max_iters_long", C.c_int32),
                ("tol", C.c_double), ("beta0", C.c_double), ("same_chain_eps", C.c_double), ("ray_eps", C.c_double),
                ("seed", C.c_uint64), ("walk_id_base", C.c_uint64), ("recip_repeats", C.c_int32),
                ("selective", C.c_int32)]


class WalkOut(C.Structure):
    _fields_ = [("status", C.c_int32), ("iters", C.c_int32), ("trials", C.c_uint32), ("truncated", C.c_int32),
                ("G", C.c_double), ("T", C.c_double), ("kappa", C.c_double), ("w", C.c_double),
                ("pos", (C.c_double * 3) * KMAX), ("prim", C.c_int32 * KMAX), ("surf", C.c_int32 * KMAX),
                ("xL", C.c_double * 3), ("pdfL", C.c_double), ("target", C.c_float * 3), ("bin", C.c_int32),
                ("total_iters", C.c_int64), ("attempts", C.c_int64), ("k", C.c_int32), ("tau", C.c_uint32),
                ("Pn", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        dp = C.POINTER(C.c_double)
        _lib.orc_scene_create.restype = P
        _lib.orc_scene_create.argtypes = [C.POINTER(Surface), C.c_int, P, P, C.c_int, P, P, C.c_int,
                                          C.POINTER(Light), C.c_int]
        _lib.orc_scene_destroy.argtypes = [P]
        _lib.orc_scene_extent.restype = C.c_double
        _lib.orc_scene_extent.argtypes = [P]
        _lib.orc_walks.argtypes = [P, C.POINTER(SeedCfg), C.POINTER(Opts), P, P, C.c_int32, P, C.c_int64,
                                   C.POINTER(WalkOut)]
        _lib.orc_closest.restype = C.c_int
        _lib.orc_closest.argtypes = [P, dp, dp, C.c_double, C.c_double, C.c_int, C.c_int, dp,
                                     C.POINTER(C.c_int32), dp]
        _lib.orc_constraint.restype = C.c_int
        _lib.orc_constraint.argtypes = [P, C.c_int, C.c_uint32, dp, dp, dp, P, P, dp, dp]
        _lib.orc_newton_chain.restype = C.c_int
        _lib.orc_newton_chain.argtypes = [P, C.POINTER(Opts), C.c_int, C.c_uint32, dp, dp, dp, P, P,
                                          C.POINTER(C.c_int32), dp]
        _lib.orc_walk_from_target.restype = C.c_int
        _lib.orc_walk_from_target.argtypes = [P, C.POINTER(Opts), C.c_int, C.c_uint32, C.c_int, dp, dp, dp, dp, dp,
                                              P, P, C.POINTER(C.c_int32), dp, dp]
        _lib.orc_ggt.restype = C.c_double
        _lib.orc_ggt.argtypes = [P, C.POINTER(Opts), C.c_int, C.c_double, C.c_int, C.c_uint32, C.c_int, dp, dp, dp,
                                 dp, P, P]
        _lib.orc_kappa.restype = C.c_double
        _lib.orc_kappa.argtypes = [P, C.c_int, C.c_uint32, dp, dp, dp, P, P]
        _lib.orc_seed.restype = C.c_int
        _lib.orc_seed.argtypes = [P, C.POINTER(SeedCfg), C.POINTER(Opts), P, C.c_int32, C.c_int64, C.c_uint32,
                                  C.POINTER(C.c_float), dp, C.POINTER(C.c_float), C.POINTER(C.c_int32)]
        _lib.orc_fresnel.restype = C.c_double
        _lib.orc_fresnel.argtypes = [C.c_double, C.c_double, C.c_double]
        _lib.orc_philox.argtypes = [P, P, P]
        _lib.orc_philox_batch.argtypes = [P, C.c_int64, P, P]
        _lib.orc_guide_tables.argtypes = [P, C.c_int, C.c_int, P]
        _lib.orc_walk_trace.restype = C.c_int
        _lib.orc_walk_trace.argtypes = [P, C.POINTER(Opts), C.c_int, C.c_uint32, dp, dp, dp, dp, dp,
                                        C.POINTER(C.c_int32)]
        _lib.orc_accumulate.argtypes = [C.POINTER(SeedCfg), P, C.c_int32, C.c_int64, P, P, P, P]
        _lib.orc_seed_ex.restype = C.c_int
        _lib.orc_seed_ex.argtypes = [P, C.POINTER(SeedCfg), C.POINTER(Opts), P, C.c_int32, C.c_int64, C.c_uint32,
                                     P, P, P, P, P, P, P]
        _lib.orc_guide_dir_tables.argtypes = [P, C.c_int, C.c_int, P, P, P]
        _lib.orc_accumulate_dir.argtypes = [C.POINTER(SeedCfg), P, C.c_int32, C.c_int64, P, P, P, P, P, P]
        _lib.orc_tangent_basis.argtypes = [P, C.c_int32, C.c_int32, dp, dp, dp]
        _lib.orc_stree_build.restype = P
        _lib.orc_stree_build.argtypes = [P, C.c_int64, C.c_float, C.c_float, C.c_int32, C.c_float, C.c_float]
        _lib.orc_stree_free.argtypes = [P]
        _lib.orc_stree_info.argtypes = [P, P]
        _lib.orc_stree_get.argtypes = [P] + [P] * 11
        _lib.orc_record_samples.argtypes = [P, C.c_int32, C.c_int64, P, P, P, P, P, P, P, P, C.c_float, P]
        _lib.orc_vmf_sample.argtypes = [P, C.c_float, C.c_float, C.c_float, P]
        _lib.orc_trace_photons.argtypes = [P, C.POINTER(PhotonDesc), C.c_int64, C.c_int64, P, P, P, P, P]
        _lib.orc_training_schedule.restype = C.c_int
        _lib.orc_training_schedule.argtypes = [C.c_int64, C.c_double, P, C.c_int32, P]
        _lib.orc_set_offset_uv.argtypes = [P, C.c_int]
        _lib.orc_scatter.restype = C.c_int
        _lib.orc_scatter.argtypes = [C.c_int, C.c_double, C.c_double, dp, dp, dp]
    return _lib


def _d3(v):
    return (C.c_double * 3)(*[float(x) for x in v])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def philox(ctr: np.ndarray, key) -> np.ndarray:
    """Philox4x32-10 on counters ctr [n,4] u32 with key (k0,k1)."""
    L = lib()
    ctr = np.ascontiguousarray(ctr, np.uint32)
    out = np.zeros_like(ctr)
    k = np.asarray(key, np.uint32)
    L.orc_philox_batch(_ptr(ctr), C.c_int64(ctr.shape[0]), _ptr(k), _ptr(out))
    return out


def training_schedule(budget, train_frac=0.3):
    """The paper's training schedule, simulated pass by pass: (iterations, render)."""
    it = np.zeros(64, np.int64)
    r = np.zeros(1, np.int64)
    m = lib().orc_training_schedule(int(budget), float(train_frac), _ptr(it), 64, _ptr(r))
    assert m >= 0
    return [int(x) for x in it[:m]], int(r[0])


def set_offset_uv(uv=None):
    """Offset-normal uniforms (u1, u2 per vertex, [k, 2]) used by the explicit-chain entry points
    (constraint, newton_chain, walk_from_target, ggt, kappa) on glossy surfaces [R37]; None = 0."""
    if uv is None:
        lib().orc_set_offset_uv(None, 0)
        return
    a = np.ascontiguousarray(uv, np.float64).reshape(-1)
    lib().orc_set_offset_uv(a.ctypes.data_as(C.c_void_p), a.size // 2)


def fresnel(cos_i, eta1, eta2) -> float:
    return lib().orc_fresnel(float(cos_i), float(eta1), float(eta2))


def scatter(isT, eta1, eta2, d, n):
    out = (C.c_double * 3)()
    ok = lib().orc_scatter(int(isT), float(eta1), float(eta2), _d3(d), _d3(n), out)
    return (np.array(out[:]) if ok else None)


def guide_tables(E: np.ndarray) -> np.ndarray:
    """Inclusive prefix sums of the defensive integer weights W' per cell."""
    E = np.ascontiguousarray(E, np.float32)
    prefix = np.zeros(E.shape, np.uint64)
    lib().orc_guide_tables(_ptr(E), int(E.shape[0]), int(E.shape[1]), _ptr(prefix))
    return prefix


def guide_dir_tables(H: np.ndarray):
    """configs[4] tables from a typed direction histogram H [cells, 126, bins]."""
    H = np.ascontiguousarray(H, np.float32)
    nc, nt, nb = H.shape
    assert nt == 126
    npf = np.zeros((nc, 6), np.uint64)
    tpf = np.zeros((nc, 126), np.uint64)
    dpf = np.zeros((nc, 126, nb), np.uint32)
    lib().orc_guide_dir_tables(_ptr(H), nc, nb, _ptr(npf), _ptr(tpf), _ptr(dpf))
    return npf, tpf, dpf


FLT_MAX = float(np.finfo(np.float32).max)
# Eq. 12 (kappa = sigma'^-2) unclamped; KAPPA_CLAMP_R30B is the measured product option
STREE_DEFAULTS = dict(eps=0.1, c_thr=1.0, max_depth=32, kappa_min=0.0, kappa_max=FLT_MAX)
KAPPA_CLAMP_R30B = (1.0, 300.0)


def stree_build(records: np.ndarray, eps=0.1, c_thr=1.0, max_depth=32, kappa_min=0.0, kappa_max=FLT_MAX) -> dict:
    """STree + vMF guide from sample records (GSAMPLE array): tree, leaf lists, lobes, tables."""
    L = lib()
    rec = np.ascontiguousarray(records, GSAMPLE)
    h = L.orc_stree_build(_ptr(rec), rec.shape[0], eps, c_thr, max_depth, kappa_min, kappa_max)
    info = np.zeros(6, np.int64)
    L.orc_stree_info(h, _ptr(info))
    nn, nl, root, thr, nv, nlobe = (int(x) for x in info)
    out = dict(n_nodes=nn, n_leaves=nl, root_ref=root, thr=thr, n_valid=nv, n_lobes=nlobe,
               nodes=np.zeros(max(nn, 1), SNODE), leaf_begin=np.zeros(nl, np.int64), leaf_count=np.zeros(nl, np.int64),
               leaf_ids=np.zeros(max(nlobe, 1), np.int64), grp_off=np.zeros((nl, 127), np.int32),
               lobe_sample=np.zeros(max(nlobe, 1), np.int64), lobe_prefix=np.zeros(max(nlobe, 1), np.uint64),
               lobe_mu=np.zeros((max(nlobe, 1), 4), np.float32), n_prefix=np.zeros((nl, 6), np.uint64),
               type_prefix=np.zeros((nl, 126), np.uint64), leaf_own=np.zeros(max(nl, 1), np.int64))
    L.orc_stree_get(h, *(_ptr(out[k]) for k in ("nodes", "leaf_begin", "leaf_count", "leaf_ids", "grp_off",
                                                "lobe_sample", "lobe_prefix", "lobe_mu", "n_prefix", "type_prefix",
                                                "leaf_own")))
    L.orc_stree_free(h)
    out["nodes"] = out["nodes"][:nn]
    for k in ("leaf_ids", "lobe_sample", "lobe_prefix", "lobe_mu"):
        out[k] = out[k][:nlobe]
    return out


def record_samples(xD, spp, status, w, x1, k, tau, xL, wv=None, nD=None, alpha=0.0) -> np.ndarray:
    """Sample records (GSAMPLE) of one iteration's walks (Eq. 9 samples); with wv / nD (per
    receiver) the weights carry a GGX(alpha) glossy separator (Eq. 14, R35)."""
    n = len(status)
    out = np.zeros(n, GSAMPLE)
    arrs = [np.ascontiguousarray(a, dt) for a, dt in ((xD, np.float32), (status, np.int32), (w, np.float32),
                                                      (x1, np.float32), (k, np.int32), (tau, np.uint32),
                                                      (xL, np.float32))]
    g = [None, None] if wv is None else [np.ascontiguousarray(wv, np.float32), np.ascontiguousarray(nD, np.float32)]
    lib().orc_record_samples(_ptr(arrs[0]), int(spp), n, *(_ptr(a) for a in arrs[1:]),
                             _ptr(g[0]) if g[0] is not None else None, _ptr(g[1]) if g[1] is not None else None,
                             float(alpha), _ptr(out))
    return out


def vmf_sample(mu, kappa, u1, u2) -> np.ndarray:
    mu = np.ascontiguousarray(mu, np.float32)
    out = np.zeros(3, np.float32)
    lib().orc_vmf_sample(_ptr(mu), float(kappa), float(u1), float(u2), _ptr(out))
    return out


def make_opts(w, **over) -> Opts:
    o = w.opts
    d = dict(max_iters=o.max_iters, trials=o.trials, k_max=o.k_max, tol=o.tol, beta0=o.beta0, seed=o.seed,
             walk_id_base=o.walk_id_base, same_chain_eps=0.0, ray_eps=0.0,
             max_iters_long=getattr(o, "max_iters_long", 0), recip_repeats=getattr(o, "recip_repeats", 1),
             selective=int(bool(o.flags & 16)))
    d.update(over)
    r = Opts()
    for k, v in d.items():
        setattr(r, k, v)
    return r


class OracleScene:
    """The oracle's own copy of a workload's scene (fp64 + its median-split BVH)."""

    def __init__(self, w):
        L = lib()
        self.w = w
        pos, nrm, idx, ts, ranges = w.mesh_arrays()
        self._keep = [pos, nrm, idx, ts]
        S = (Surface * max(1, len(w.surfaces)))()
        for i, s in enumerate(w.surfaces):
            S[i].kind, S[i].mat = s.kind, s.mat
            S[i].tri_begin, S[i].tri_count = ranges[i]
            S[i].eta_in, S[i].eta_out, S[i].reflectance, S[i].radius = s.eta_in, s.eta_out, s.reflectance, s.radius
            S[i].center[:] = list(s.center)
            S[i].origin[:] = list(s.origin)
            S[i].edge_u[:] = list(s.edge_u)
            S[i].edge_v[:] = list(s.edge_v)
            S[i].roughness = float(getattr(s, "roughness", 0.0))
        Ls = (Light * max(1, len(w.lights)))()
        for i, l in enumerate(w.lights):
            Ls[i].kind, Ls[i].emit = l.kind, l.emit
            Ls[i].position[:] = list(l.position)
            Ls[i].edge_u[:] = list(l.edge_u)
            Ls[i].edge_v[:] = list(l.edge_v)
        self._S, self._L = S, Ls
        self.h = L.orc_scene_create(S, len(w.surfaces), _ptr(pos), _ptr(nrm), pos.shape[0], _ptr(idx), _ptr(ts),
                                    idx.shape[0], Ls, len(w.lights))
        self.extent = L.orc_scene_extent(self.h)
        self.prefix = None
        self.cfg = self._seed_cfg()

    def __del__(self):
        try:
            lib().orc_scene_destroy(self.h)
        except Exception:
            pass

    def _seed_cfg(self) -> SeedCfg:
        s = self.w.seed
        c = SeedCfg()
        c.mode, c.surf_id, c.k, c.tau = s.mode, s.surf_id, s.k, s.tau
        c.grid_origin[:] = list(s.grid_origin)
        c.grid_extent[:] = list(s.grid_extent)
        c.cells_x, c.cells_y, c.bins_x, c.bins_y = s.cells_x, s.cells_y, s.bins_x, s.bins_y
        c.uv_origin[:] = list(s.uv_origin)
        c.uv_scale[:] = list(s.uv_scale)
        c.uv_plane_y = s.uv_plane_y
        if s.mode == 3:
            nb = s.bins_x * s.bins_y
            self.set_dir_hist(np.zeros((s.cells_x * s.cells_y, 126, nb), np.float32), c)
        elif s.mode == 4:                      # STree + vMF guide: empty tree (learned branch absent)
            self.set_stree(stree_build(np.zeros(0, GSAMPLE)), c)
        elif self.w.energies is not None:
            self.set_energies(self.w.energies, c)
        return c

    def set_dir_hist(self, H, c=None):
        """configs[4]: build the typed tables from histogram H [cells,126,bins] (zeros = reset)."""
        c = c or self.cfg
        self.dir_tables = guide_dir_tables(H)
        npf, tpf, dpf = self.dir_tables
        c.n_prefix, c.type_prefix, c.dir_prefix = _ptr(npf), _ptr(tpf), _ptr(dpf)

    def set_stree(self, G: dict, c=None):
        """Seed mode 4: sample from an STree + vMF guide (stree_build output)."""
        c = c or self.cfg
        self.stree = G
        c.mode = 4
        c.root_ref = G["root_ref"]
        c.nodes, c.grp_off = _ptr(G["nodes"]), _ptr(G["grp_off"])
        c.lobe_prefix, c.lobe_mu = _ptr(G["lobe_prefix"]), _ptr(G["lobe_mu"])
        c.n_prefix, c.type_prefix = _ptr(G["n_prefix"]), _ptr(G["type_prefix"])
        c.leaf_own = _ptr(G["leaf_own"])

    def trace_photons(self, n_photons, plane_point, plane_normal, first=0, count=None, seed=0, base=0,
                      max_vertices=6):
        """Photon records (GSAMPLE) of photons first..first+count of an N = n_photons run, plus
        per photon: vertex count, vertices / prims / surfs in x_D order."""
        count = n_photons - first if count is None else count
        d = PhotonDesc(n_photons=n_photons, seed=seed, photon_id_base=base, max_vertices=max_vertices, ray_eps=0.0)
        d.plane_point[:] = [float(v) for v in plane_point]
        d.plane_normal[:] = [float(v) for v in plane_normal]
        rec = np.zeros(count, GSAMPLE)
        nv = np.zeros(count, np.int32)
        verts = np.zeros((count, KMAX, 3), np.float64)
        prims = np.zeros((count, KMAX), np.int32)
        surfs = np.zeros((count, KMAX), np.int32)
        lib().orc_trace_photons(self.h, C.byref(d), first, count, _ptr(rec), _ptr(nv), _ptr(verts), _ptr(prims),
                                _ptr(surfs))
        return rec, nv, verts, prims, surfs

    def set_energies(self, E, c=None):
        c = c or self.cfg
        self.prefix = guide_tables(E)
        c.prefix = self.prefix.ctypes.data_as(C.POINTER(C.c_uint64))

    def opts(self, **over) -> Opts:
        return make_opts(self.w, **over)

    def walks(self, walk_ids, opts: Opts = None):
        """Run the walk (primary + trials) for explicit walk indices."""
        opts = opts or self.opts()
        ids = np.ascontiguousarray(walk_ids, np.int64)
        out = (WalkOut * max(1, ids.shape[0]))()
        w = self.w
        lib().orc_walks(self.h, C.byref(self.cfg), C.byref(opts), _ptr(w.xD), _ptr(w.nD), w.spp, _ptr(ids),
                        ids.shape[0], out)
        n = ids.shape[0]
        k = w.seed.k
        raw = np.frombuffer(out, dtype=np.dtype(_np_walkout()), count=n)
        res = {f: raw[f].copy() for f in raw.dtype.names}
        res["pos"] = res["pos"][:, :k]
        res["prim"] = res["prim"][:, :k]
        res["surf"] = res["surf"][:, :k]
        res["walk"] = ids
        return res

    def closest(self, o, d, tmin=1e-9, tmax=1e300, spec_only=True, use_bvh=True):
        t = C.c_double()
        prim = C.c_int32()
        p = (C.c_double * 3)()
        s = lib().orc_closest(self.h, _d3(o), _d3(d), tmin, tmax, int(spec_only), int(use_bvh), C.byref(t),
                              C.byref(prim), p)
        return s, t.value, prim.value, np.array(p[:])

    def constraint(self, k, tau, xD, xL, pos, prim, surf):
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
        prim = np.ascontiguousarray(prim, np.int32)
        surf = np.ascontiguousarray(surf, np.int32)
        Cv = (C.c_double * (2 * k))()
        J = (C.c_double * (4 * k * k))()
        ok = lib().orc_constraint(self.h, k, tau, _d3(xD), _d3(xL), pos.ctypes.data_as(C.POINTER(C.c_double)),
                                  _ptr(prim), _ptr(surf), Cv, J)
        return ok, np.array(Cv[:]), np.array(J[:]).reshape(2 * k, 2 * k)

    def newton_chain(self, k, tau, xD, xL, pos, prim, surf, opts=None):
        opts = opts or self.opts()
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1).copy()
        prim = np.ascontiguousarray(prim, np.int32).copy()
        surf = np.ascontiguousarray(surf, np.int32).copy()
        it = C.c_int32()
        hist = np.zeros(opts.max_iters + 2, np.float64)
        st = lib().orc_newton_chain(self.h, C.byref(opts), k, tau, _d3(xD), _d3(xL),
                                    pos.ctypes.data_as(C.POINTER(C.c_double)), _ptr(prim), _ptr(surf), C.byref(it),
                                    hist.ctypes.data_as(C.POINTER(C.c_double)))
        return st, it.value, pos.reshape(k, 3), prim, surf, hist[:it.value + 1]

    def walk_from_target(self, xD, nD, xL, target, light_id=0, opts=None, k=None, tau=None):
        opts = opts or self.opts()
        k = self.w.seed.k if k is None else k
        tau = self.w.seed.tau if tau is None else tau
        pos = np.zeros(3 * k, np.float64)
        prim = np.zeros(k, np.int32)
        surf = np.zeros(k, np.int32)
        it = C.c_int32()
        G = C.c_double()
        T = C.c_double()
        st = lib().orc_walk_from_target(self.h, C.byref(opts), k, tau, light_id, _d3(xD), _d3(nD), _d3(xL),
                                        _d3(target), pos.ctypes.data_as(C.POINTER(C.c_double)), _ptr(prim),
                                        _ptr(surf), C.byref(it), C.byref(G), C.byref(T))
        return dict(status=st, iters=it.value, pos=pos.reshape(k, 3), prim=prim, surf=surf, G=G.value, T=T.value)

    def ggt(self, k, tau, xD, nD, xL, pos, prim, surf, method=0, delta=1e-5, light_id=0, opts=None):
        opts = opts or self.opts()
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
        prim = np.ascontiguousarray(prim, np.int32)
        surf = np.ascontiguousarray(surf, np.int32)
        return lib().orc_ggt(self.h, C.byref(opts), method, delta, k, tau, light_id, _d3(xD), _d3(nD), _d3(xL),
                             pos.ctypes.data_as(C.POINTER(C.c_double)), _ptr(prim), _ptr(surf))

    def walk_trace(self, xD, xL, target, opts=None):
        opts = opts or self.opts()
        res = np.zeros(opts.max_iters + 2)
        beta = np.zeros(opts.max_iters + 2)
        it = C.c_int32()
        st = lib().orc_walk_trace(self.h, C.byref(opts), self.w.seed.k, self.w.seed.tau, _d3(xD), _d3(xL),
                                  _d3(target), res.ctypes.data_as(C.POINTER(C.c_double)),
                                  beta.ctypes.data_as(C.POINTER(C.c_double)), C.byref(it))
        return st, it.value, res[:it.value + 1], beta[:it.value + 1]

    def accumulate(self, status, w, x1):
        """Guide histogram [cells][bins] (fp64) from per-walk status, w and x_1* (float [n,3])."""
        sp = self.w.seed
        hist = np.zeros((sp.cells_x * sp.cells_y, sp.bins_x * sp.bins_y), np.float64)
        st = np.ascontiguousarray(status, np.int32)
        wv = np.ascontiguousarray(w, np.float32)
        x1 = np.ascontiguousarray(x1, np.float32)
        lib().orc_accumulate(C.byref(self.cfg), _ptr(self.w.xD), self.w.spp, st.shape[0], _ptr(st), _ptr(wv),
                             _ptr(x1), _ptr(hist))
        return hist

    def seed_ex(self, walk, trial=0, opts=None):
        opts = opts or self.opts()
        tgt = np.zeros(3, np.float32)
        b, n, learned = (np.zeros(1, np.int32) for _ in range(3))
        tau, ib = np.zeros(1, np.uint32), np.zeros(1, np.uint32)
        pn = np.zeros(1, np.float64)
        ok = lib().orc_seed_ex(self.h, C.byref(self.cfg), C.byref(opts), _ptr(self.w.xD), self.w.spp, int(walk),
                               int(trial), _ptr(tgt), _ptr(b), _ptr(n), _ptr(tau), _ptr(learned), _ptr(ib), _ptr(pn))
        return dict(ok=ok, target=tgt, bin=int(b[0]), n=int(n[0]), tau=int(tau[0]), learned=int(learned[0]),
                    init_bits=int(ib[0]), Pn=float(pn[0]))

    def accumulate_dir(self, status, w, x1, k, tau):
        sp = self.w.seed
        hist = np.zeros((sp.cells_x * sp.cells_y, 126, sp.bins_x * sp.bins_y), np.float64)
        st = np.ascontiguousarray(status, np.int32)
        wv = np.ascontiguousarray(w, np.float32)
        x1 = np.ascontiguousarray(x1, np.float32)
        kk = np.ascontiguousarray(k, np.int32)
        tt = np.ascontiguousarray(tau, np.uint32)
        lib().orc_accumulate_dir(C.byref(self.cfg), _ptr(self.w.xD), self.w.spp, st.shape[0], _ptr(st), _ptr(wv),
                                 _ptr(x1), _ptr(kk), _ptr(tt), _ptr(hist))
        return hist

    def tangent_basis(self, prim, surf, p):
        a = (C.c_double * 3)()
        b = (C.c_double * 3)()
        lib().orc_tangent_basis(self.h, int(prim), int(surf), _d3(p), a, b)
        return np.array(a[:]), np.array(b[:])

    def kappa(self, k, tau, xD, xL, pos, prim, surf):
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1)
        prim = np.ascontiguousarray(prim, np.int32)
        surf = np.ascontiguousarray(surf, np.int32)
        return lib().orc_kappa(self.h, k, tau, _d3(xD), _d3(xL), pos.ctypes.data_as(C.POINTER(C.c_double)),
                               _ptr(prim), _ptr(surf))

    def seed(self, walk, trial=0, opts=None):
        opts = opts or self.opts()
        xL = (C.c_float * 3)()
        tgt = (C.c_float * 3)()
        pdf = C.c_double()
        b = C.c_int32()
        ok = lib().orc_seed(self.h, C.byref(self.cfg), C.byref(opts), _ptr(self.w.xD), self.w.spp, int(walk),
                            int(trial), xL, C.byref(pdf), tgt, C.byref(b))
        return ok, np.array(xL[:], np.float32), pdf.value, np.array(tgt[:], np.float32), b.value


def _np_walkout():
    return np.dtype([("status", np.int32), ("iters", np.int32), ("trials", np.uint32), ("truncated", np.int32),
                     ("G", np.float64), ("T", np.float64), ("kappa", np.float64), ("w", np.float64),
                     ("pos", np.float64, (KMAX, 3)), ("prim", np.int32, (KMAX,)), ("surf", np.int32, (KMAX,)),
                     ("xL", np.float64, (3,)), ("pdfL", np.float64), ("target", np.float32, (3,)), ("bin", np.int32),
                     ("total_iters", np.int64), ("attempts", np.int64), ("k", np.int32), ("tau", np.uint32),
                     ("Pn", np.float64)])
