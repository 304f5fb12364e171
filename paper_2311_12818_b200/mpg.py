"""Thin ctypes binding of libmpg.so (include/mpg.h).

Argument marshalling only: every step of the walk runs in the CUDA kernels of
csrc/.  PyTorch provides device memory and streams.  There is no CPU fallback:
if the shared library is missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPG_LIB", os.path.join(HERE, "libmpg.so"))   # MPG_LIB: experiment variants
KMAX = 8
FLT_MAX = float(np.finfo(np.float32).max)   # unclamped vMF concentration (Eq. 12, R30)
KAPPA_CLAMP_R30B = (1.0, 300.0)             # the measured product option (R30b)
STATUS_NAMES = ["CONVERGED", "MAXITER", "SEED_FAIL", "BAD_SIDE", "DEGENERATE", "OCCLUDED", "INACTIVE"]


class MPGError(RuntimeError):
    pass


# ----------------------------------------------------------------------------
# C records (same layout as include/mpg.h)
# ----------------------------------------------------------------------------
class mpg_surface_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mat", C.c_int32), ("eta_in", C.c_float), ("eta_out", C.c_float),
                ("reflectance", C.c_float), ("center", C.c_float * 3), ("radius", C.c_float),
                ("origin", C.c_float * 3), ("edge_u", C.c_float * 3), ("edge_v", C.c_float * 3),
                ("positions", C.c_void_p), ("normals", C.c_void_p), ("indices", C.c_void_p),
                ("n_vertices", C.c_int32), ("n_triangles", C.c_int32), ("roughness", C.c_float)]


class mpg_light_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("emit", C.c_float), ("position", C.c_float * 3), ("edge_u", C.c_float * 3),
                ("edge_v", C.c_float * 3)]


class mpg_sampler_desc(C.Structure):
    _fields_ = [("mode", C.c_int32), ("surf_id", C.c_int32), ("k", C.c_int32), ("tau", C.c_uint32)]


class mpg_guide_desc(C.Structure):
    _fields_ = [("grid_origin", C.c_float * 2), ("grid_extent", C.c_float * 2), ("cells_x", C.c_int32),
                ("cells_y", C.c_int32), ("bins_x", C.c_int32), ("bins_y", C.c_int32), ("uv_origin", C.c_float * 2),
                ("uv_scale", C.c_float * 2), ("uv_plane_y", C.c_float), ("domain", C.c_int32), ("n_types", C.c_int32)]


class mpg_walk_opts(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("tol", C.c_float), ("beta0", C.c_float), ("trials", C.c_int32),
                ("k_max", C.c_uint32), ("same_chain_eps", C.c_float), ("ray_eps", C.c_float), ("flags", C.c_uint32),
                ("seed", C.c_uint64), ("walk_id_base", C.c_uint64), ("max_iters_long", C.c_int32),
                ("recip_repeats", C.c_int32)]


class mpg_query(C.Structure):
    _fields_ = [("xD", C.c_void_p), ("nD", C.c_void_p), ("n_recv", C.c_int64), ("spp", C.c_int32)]


class mpg_seed_buf(C.Structure):
    _fields_ = [("xL", C.c_void_p), ("target", C.c_void_p), ("bin", C.c_void_p), ("ctype", C.c_void_p),
                ("pn", C.c_void_p)]


class mpg_walk_buf(C.Structure):
    _fields_ = [("chain", C.c_void_p), ("status", C.c_void_p), ("iters", C.c_void_p), ("G", C.c_void_p),
                ("T", C.c_void_p), ("w", C.c_void_p), ("trials", C.c_void_p), ("ctype", C.c_void_p)]


class mpg_stree_desc(C.Structure):
    _fields_ = [("max_samples", C.c_int64), ("eps", C.c_float), ("c_thr", C.c_float), ("kappa_min", C.c_float),
                ("kappa_max", C.c_float), ("max_depth", C.c_int32), ("keep_all", C.c_int32)]


class mpg_stree_info(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("n_nodes", "n_leaves", "root_ref", "thr", "n_valid", "n_lobes")]


class mpg_photon_desc(C.Structure):
    _fields_ = [("n_photons", C.c_int64), ("seed", C.c_uint64), ("photon_id_base", C.c_uint64),
                ("plane_point", C.c_float * 3), ("plane_normal", C.c_float * 3), ("max_vertices", C.c_int32),
                ("ray_eps", C.c_float)]


GUIDE_SAMPLE_BYTES = 48

STATS_FIELDS = ["walks", "converged", "newton_iters", "primary_iters", "attempts", "rays", "trials", "truncated",
                "node_visits", "tri_tests", "vertex_iters"]


class mpg_walk_stats(C.Structure):
    _fields_ = [(f, C.c_ulonglong) for f in STATS_FIELDS] + [("by_status", C.c_ulonglong * 8)]


class mpg_scene_info(C.Structure):
    _fields_ = [("extent", C.c_float), ("n_surf", C.c_int32), ("n_light", C.c_int32), ("n_tri", C.c_int32),
                ("n_nodes", C.c_int32), ("bvh_width", C.c_int32), ("device_bytes", C.c_size_t)]


EXPORTS = ["mpg_scene_create", "mpg_scene_destroy", "mpg_scene_get_info", "mpg_trace_rays", "mpg_guide_create",
           "mpg_guide_set_histogram",
           "mpg_guide_destroy", "mpg_guide_upload", "mpg_guide_reset", "mpg_guide_accumulate", "mpg_guide_rebuild",
           "mpg_guide_download", "mpg_guide_download_dir_tables", "mpg_sample_seeds", "mpg_walk_workspace_size", "mpg_manifold_walk", "mpg_estimate",
           "mpg_debug_trace", "mpg_last_error", "mpg_version", "mpg_kernel_launches", "mpg_guide_create_stree",
           "mpg_guide_record_samples", "mpg_guide_set_samples", "mpg_guide_get_samples", "mpg_guide_stree_info",
           "mpg_guide_download_stree", "mpg_trace_photons", "mpg_splat", "mpg_guide_set_separator", "mpg_measure_fp32_peak",
           "mpg_training_schedule"]

_lib = None


def lib():
    """Load libmpg.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MPGError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        st = C.c_int
        sig = {
            "mpg_scene_create": (st, [C.POINTER(mpg_surface_desc), C.c_int32, C.POINTER(mpg_light_desc), C.c_int32, P,
                                      C.POINTER(P)]),
            "mpg_scene_destroy": (st, [P]),
            "mpg_scene_get_info": (st, [P, C.POINTER(mpg_scene_info)]),
            "mpg_trace_rays": (st, [P, P, P, C.c_int64, C.c_float, C.c_int32, P, P, P, P]),
            "mpg_guide_create": (st, [C.POINTER(mpg_guide_desc), C.POINTER(P)]),
            "mpg_guide_destroy": (st, [P]),
            "mpg_guide_upload": (st, [P, P, P]),
            "mpg_guide_reset": (st, [P, P]),
            "mpg_guide_accumulate": (st, [P, C.POINTER(mpg_query), C.POINTER(mpg_walk_buf), C.c_int64, P]),
            "mpg_guide_rebuild": (st, [P, P]),
            "mpg_guide_download": (st, [P, P, P, P]),
            "mpg_guide_set_histogram": (st, [P, P, P]),
            "mpg_guide_download_dir_tables": (st, [P, P, P, P, P]),
            "mpg_sample_seeds": (st, [P, P, C.POINTER(mpg_sampler_desc), C.POINTER(mpg_query),
                                      C.POINTER(mpg_walk_opts), C.POINTER(mpg_seed_buf), P]),
            "mpg_walk_workspace_size": (C.c_size_t, [C.c_int64, C.POINTER(mpg_sampler_desc), C.POINTER(mpg_walk_opts)]),
            "mpg_manifold_walk": (st, [P, P, C.POINTER(mpg_sampler_desc), C.POINTER(mpg_query),
                                       C.POINTER(mpg_seed_buf), C.POINTER(mpg_walk_opts), C.POINTER(mpg_walk_buf), P,
                                       P, C.c_size_t, P]),
            "mpg_estimate": (st, [P, C.c_int64, C.c_int32, P, P, P]),
            "mpg_debug_trace": (st, [P, C.c_int64, C.c_int32]),
            "mpg_last_error": (C.c_char_p, []),
            "mpg_version": (C.c_int32, []),
            "mpg_kernel_launches": (C.c_uint64, []),
            "mpg_measure_fp32_peak": (st, [C.c_int32, C.c_int32, C.POINTER(C.c_double), P]),
            "mpg_training_schedule": (st, [C.c_int64, C.c_double, P, C.c_int32, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int64)]),
            "mpg_guide_create_stree": (st, [C.POINTER(mpg_stree_desc), C.POINTER(P)]),
            "mpg_guide_record_samples": (st, [P, C.POINTER(mpg_query), C.POINTER(mpg_seed_buf),
                                              C.POINTER(mpg_walk_buf), C.c_int64, P]),
            "mpg_guide_set_samples": (st, [P, P, C.c_int64, P]),
            "mpg_guide_get_samples": (st, [P, P, C.POINTER(C.c_int64), P]),
            "mpg_guide_stree_info": (st, [P, C.POINTER(mpg_stree_info)]),
            "mpg_trace_photons": (st, [P, C.POINTER(mpg_photon_desc), P, P]),
            "mpg_splat": (st, [P, C.c_int64, C.c_int32, P, P, P]),
            "mpg_guide_set_separator": (st, [P, P, P, C.c_float]),
            "mpg_guide_download_stree": (st, [P] + [P] * 11 + [P]),
        }
        for name, (res, args) in sig.items():
            if "MPG_LIB" in os.environ and not hasattr(L, name):
                continue      # an older experiment build (tools/minb_sweep.sh) lacks newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        msg = lib().mpg_last_error().decode()
        raise MPGError(f"{what} failed ({status}): {msg}")


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


# ----------------------------------------------------------------------------
# same-named Python entry points
# ----------------------------------------------------------------------------
def mpg_scene_create(surfaces, lights, stream=None):
    n = len(surfaces)
    S = (mpg_surface_desc * n)(*surfaces)
    Ls = (mpg_light_desc * len(lights))(*lights)
    h = C.c_void_p()
    _check(lib().mpg_scene_create(S, n, Ls, len(lights), _stream_ptr(stream), C.byref(h)), "mpg_scene_create")
    return h


def mpg_scene_destroy(h):
    _check(lib().mpg_scene_destroy(h), "mpg_scene_destroy")


def mpg_scene_get_info(h) -> mpg_scene_info:
    info = mpg_scene_info()
    _check(lib().mpg_scene_get_info(h, C.byref(info)), "mpg_scene_get_info")
    return info


def mpg_trace_rays(h, orig, direc, tmin, spec_only, t, prim, surf, stream=None):
    _check(lib().mpg_trace_rays(h, _ptr(orig), _ptr(direc), orig.shape[0], tmin, int(spec_only), _ptr(t), _ptr(prim),
                                _ptr(surf), _stream_ptr(stream)), "mpg_trace_rays")


def mpg_guide_create(desc: mpg_guide_desc):
    h = C.c_void_p()
    _check(lib().mpg_guide_create(C.byref(desc), C.byref(h)), "mpg_guide_create")
    return h


def mpg_guide_destroy(h):
    _check(lib().mpg_guide_destroy(h), "mpg_guide_destroy")


def mpg_guide_upload(h, energy, stream=None):
    _check(lib().mpg_guide_upload(h, _ptr(energy), _stream_ptr(stream)), "mpg_guide_upload")


def mpg_guide_reset(h, stream=None):
    _check(lib().mpg_guide_reset(h, _stream_ptr(stream)), "mpg_guide_reset")


def mpg_guide_accumulate(h, query: mpg_query, walks: mpg_walk_buf, n: int, stream=None):
    _check(lib().mpg_guide_accumulate(h, C.byref(query), C.byref(walks), n, _stream_ptr(stream)),
           "mpg_guide_accumulate")


def mpg_guide_rebuild(h, stream=None):
    _check(lib().mpg_guide_rebuild(h, _stream_ptr(stream)), "mpg_guide_rebuild")


def mpg_guide_download(h, energy=None, prefix=None, stream=None):
    _check(lib().mpg_guide_download(h, _ptr(energy), _ptr(prefix), _stream_ptr(stream)), "mpg_guide_download")


def mpg_guide_set_histogram(h, energy, stream=None):
    _check(lib().mpg_guide_set_histogram(h, _ptr(energy), _stream_ptr(stream)), "mpg_guide_set_histogram")


def mpg_guide_download_dir_tables(h, n_prefix=None, type_prefix=None, dir_prefix=None, stream=None):
    _check(lib().mpg_guide_download_dir_tables(h, _ptr(n_prefix), _ptr(type_prefix), _ptr(dir_prefix),
                                               _stream_ptr(stream)), "mpg_guide_download_dir_tables")


def mpg_guide_create_stree(desc: mpg_stree_desc):
    h = C.c_void_p()
    _check(lib().mpg_guide_create_stree(C.byref(desc), C.byref(h)), "mpg_guide_create_stree")
    return h


def mpg_guide_record_samples(h, query, seeds, walks, n, stream=None):
    _check(lib().mpg_guide_record_samples(h, C.byref(query), C.byref(seeds), C.byref(walks), n, _stream_ptr(stream)),
           "mpg_guide_record_samples")


def mpg_guide_set_separator(h, wv=None, nD=None, alpha=0.0):
    """Glossy separator (Eq. 14): wv, nD device float32 [n_recv, 4]; None = diffuse."""
    _check(lib().mpg_guide_set_separator(h, _ptr(wv), _ptr(nD), float(alpha)), "mpg_guide_set_separator")


def mpg_guide_set_samples(h, records, n, stream=None):
    """records: device uint8 tensor of n*48 bytes (mpg_guide_sample)."""
    _check(lib().mpg_guide_set_samples(h, _ptr(records), n, _stream_ptr(stream)), "mpg_guide_set_samples")


def mpg_guide_get_samples(h, records=None, stream=None) -> int:
    n = C.c_int64(records.numel() // GUIDE_SAMPLE_BYTES if records is not None else 0)
    _check(lib().mpg_guide_get_samples(h, _ptr(records), C.byref(n), _stream_ptr(stream)), "mpg_guide_get_samples")
    return int(n.value)


def mpg_guide_stree_info(h) -> dict:
    info = mpg_stree_info()
    _check(lib().mpg_guide_stree_info(h, C.byref(info)), "mpg_guide_stree_info")
    return {f: int(getattr(info, f)) for f, _ in mpg_stree_info._fields_}


def mpg_guide_download_stree(h, stream=None) -> dict:
    """Host (numpy) copy of the current STree + vMF guide (tests and tools)."""
    import torch
    inf = mpg_guide_stree_info(h)
    L, NL, NN = inf["n_leaves"], inf["n_lobes"], inf["n_nodes"]
    dev = dict(nodes=torch.zeros(max(NN, 1), 4, dtype=torch.int32), leaf_begin=torch.zeros(L, dtype=torch.int64),
               leaf_count=torch.zeros(L, dtype=torch.int64), leaf_ids=torch.zeros(max(NL, 1), dtype=torch.int32),
               grp_off=torch.zeros(L, 127, dtype=torch.int32), lobe_sample=torch.zeros(max(NL, 1), dtype=torch.int32),
               lobe_prefix=torch.zeros(max(NL, 1), dtype=torch.int64), lobe_mu=torch.zeros(max(NL, 1), 4),
               n_prefix=torch.zeros(L, 6, dtype=torch.int64), type_prefix=torch.zeros(L, 126, dtype=torch.int64),
               leaf_own=torch.zeros(max(L, 1), dtype=torch.int32))
    dev = {k: v.cuda() for k, v in dev.items()}
    _check(lib().mpg_guide_download_stree(h, *(_ptr(dev[k]) for k in (
        "nodes", "leaf_begin", "leaf_count", "leaf_ids", "grp_off", "lobe_sample", "lobe_prefix", "lobe_mu",
        "n_prefix", "type_prefix", "leaf_own")), _stream_ptr(stream)), "mpg_guide_download_stree")
    torch.cuda.synchronize()
    out = dict(inf)
    for k, v in dev.items():
        a = v.cpu().numpy()
        if k in ("lobe_prefix", "n_prefix", "type_prefix"):
            a = a.view(np.uint64)
        out[k] = a
    out["nodes"] = out["nodes"][:NN]
    out["leaf_own"] = out["leaf_own"][:L]
    for k in ("leaf_ids", "lobe_sample", "lobe_prefix", "lobe_mu"):
        out[k] = out[k][:NL]
    return out


def mpg_trace_photons(scene, desc: mpg_photon_desc, records, stream=None):
    """records: device uint8 tensor of desc.n_photons * 48 bytes (mpg_guide_sample)."""
    _check(lib().mpg_trace_photons(scene, C.byref(desc), _ptr(records), _stream_ptr(stream)), "mpg_trace_photons")


def photon_init(ds, n_photons: int, plane_point, plane_normal, seed: int = 0, base: int = 0, stream=None,
                exchange=None):
    """Photon-based p_0: trace photons on the GPU and fit the STree guide from
    them (replaces the empty iteration-0 guide).  exchange(ds) (multi-process runs,
    dist.exchange_samples) gathers every rank's photon records before the fit, so all ranks
    start from the same guide.  Returns the number of landed photons (this rank's)."""
    import torch
    d = mpg_photon_desc(n_photons=n_photons, seed=seed, photon_id_base=base, max_vertices=6, ray_eps=0.0)
    d.plane_point = (C.c_float * 3)(*[float(v) for v in plane_point])
    d.plane_normal = (C.c_float * 3)(*[float(v) for v in plane_normal])
    cap = ds.stree_desc.max_samples
    rec = torch.empty(n_photons * GUIDE_SAMPLE_BYTES, dtype=torch.uint8, device="cuda")
    mpg_trace_photons(ds.h, d, rec, stream)
    landed = int((rec.view(torch.float32).view(-1, 12)[:, 9] > 0).sum())   # w > 0
    assert n_photons <= cap, "photon records exceed the STree guide's max_samples"
    mpg_guide_set_samples(ds.guide, rec, n_photons, stream)
    if exchange is not None:
        exchange(ds)
    mpg_guide_rebuild(ds.guide, stream)
    return landed


def mpg_sample_seeds(scene, guide, sampler, query, opts, seeds, stream=None):
    _check(lib().mpg_sample_seeds(scene, guide, C.byref(sampler), C.byref(query), C.byref(opts), C.byref(seeds),
                                  _stream_ptr(stream)), "mpg_sample_seeds")


def mpg_walk_workspace_size(n, sampler, opts) -> int:
    return int(lib().mpg_walk_workspace_size(n, C.byref(sampler), C.byref(opts)))


def mpg_manifold_walk(scene, guide, sampler, query, seeds, opts, out, stats, workspace, stream=None):
    _check(lib().mpg_manifold_walk(scene, guide, C.byref(sampler), C.byref(query), C.byref(seeds), C.byref(opts),
                                   C.byref(out), _ptr(stats), _ptr(workspace), workspace.numel(),
                                   _stream_ptr(stream)), "mpg_manifold_walk")


def mpg_estimate(w, n_recv, spp, mean, var=None, stream=None):
    _check(lib().mpg_estimate(_ptr(w), n_recv, spp, _ptr(mean), _ptr(var), _stream_ptr(stream)), "mpg_estimate")


def mpg_splat(w, n_recv, spp, sum_, sumsq=None, stream=None):
    _check(lib().mpg_splat(_ptr(w), n_recv, spp, _ptr(sum_), _ptr(sumsq), _stream_ptr(stream)), "mpg_splat")


def mpg_debug_trace(buf=None, n_walks=0, stride=0):
    _check(lib().mpg_debug_trace(_ptr(buf), n_walks, stride), "mpg_debug_trace")


def mpg_version() -> int:
    return int(lib().mpg_version())


def mpg_kernel_launches() -> int:
    return int(lib().mpg_kernel_launches())


def mpg_measure_fp32_peak(iters: int = 20000, reps: int = 5, stream=None) -> float:
    """Measured FP32 FFMA throughput of this GPU in TFLOP/s (bench.py's roofline peak)."""
    v = C.c_double()
    _check(lib().mpg_measure_fp32_peak(int(iters), int(reps), C.byref(v), _stream_ptr(stream)), "mpg_measure_fp32_peak")
    return float(v.value)


# ----------------------------------------------------------------------------
# convenience: a Workload (paper_2311_12818_b200.workloads) on the device
# ----------------------------------------------------------------------------
def _f3(v):
    return (C.c_float * 3)(*[float(a) for a in v])


class DeviceScene:
    """Scene + (optional) guide of a Workload, resident on the current CUDA device."""

    def __init__(self, w: "W.Workload", stream=None, stree_capacity=None, stree_kappa=(0.0, FLT_MAX)):
        import torch
        if not torch.cuda.is_available():
            raise MPGError("no CUDA device: the manifold walk has no CPU path")
        self.w = w
        descs = []
        self._keep = []
        for s in w.surfaces:
            d = mpg_surface_desc()
            d.kind, d.mat = s.kind, s.mat
            d.eta_in, d.eta_out, d.reflectance, d.radius = s.eta_in, s.eta_out, s.reflectance, s.radius
            d.roughness = float(getattr(s, "roughness", 0.0))
            d.center, d.origin, d.edge_u, d.edge_v = _f3(s.center), _f3(s.origin), _f3(s.edge_u), _f3(s.edge_v)
            if s.kind == W.SURF_MESH:
                P = np.ascontiguousarray(s.positions, np.float32)
                N = np.ascontiguousarray(s.normals, np.float32)
                I = np.ascontiguousarray(s.indices, np.int32)
                self._keep += [P, N, I]
                d.positions, d.normals, d.indices = P.ctypes.data, N.ctypes.data, I.ctypes.data
                d.n_vertices, d.n_triangles = P.shape[0], I.shape[0]
            descs.append(d)
        lights = []
        for l in w.lights:
            L = mpg_light_desc()
            L.kind, L.emit = l.kind, l.emit
            L.position, L.edge_u, L.edge_v = _f3(l.position), _f3(l.edge_u), _f3(l.edge_v)
            lights.append(L)
        self.h = mpg_scene_create(descs, lights, stream)
        self.info = mpg_scene_get_info(self.h)
        self.extent = float(self.info.extent)
        sp = w.seed
        self.sampler = mpg_sampler_desc(sp.mode, sp.surf_id, sp.k, sp.tau)
        self.guide = None
        self.stree = sp.mode == W.SEED_GUIDE_STREE
        if self.stree:
            d = mpg_stree_desc(max_samples=int(stree_capacity if stree_capacity is not None else w.n_walks),
                               eps=0.1, c_thr=1.0, kappa_min=float(stree_kappa[0]),
                               kappa_max=float(stree_kappa[1]), max_depth=32)
            self.stree_desc = d
            self.guide = mpg_guide_create_stree(d)
        elif sp.mode in (W.SEED_GUIDE_UV, W.SEED_GUIDE_DIR):
            g = mpg_guide_desc()
            g.grid_origin = (C.c_float * 2)(*sp.grid_origin)
            g.grid_extent = (C.c_float * 2)(*sp.grid_extent)
            g.cells_x, g.cells_y, g.bins_x, g.bins_y = sp.cells_x, sp.cells_y, sp.bins_x, sp.bins_y
            g.uv_origin = (C.c_float * 2)(*sp.uv_origin)
            g.uv_scale = (C.c_float * 2)(*sp.uv_scale)
            g.uv_plane_y = sp.uv_plane_y
            g.domain = 1 if sp.mode == W.SEED_GUIDE_DIR else 0
            g.n_types = sp.n_types
            self.guide_desc = g
            self.guide = mpg_guide_create(g)
            if w.energies is not None and sp.mode == W.SEED_GUIDE_UV:
                self.upload_energies(w.energies, stream)
            else:
                mpg_guide_reset(self.guide, stream)

    def upload_energies(self, E, stream=None):
        import torch
        e = torch.as_tensor(np.ascontiguousarray(E, np.float32)).cuda()
        mpg_guide_upload(self.guide, e, stream)
        torch.cuda.synchronize()

    def info_guide_size(self) -> int:
        """Floats in the guide histogram ([cells][types][bins]); 0 without a guide."""
        if self.guide is None:
            return 0
        g = self.guide_desc
        return int(g.cells_x * g.cells_y * max(1, g.n_types) * g.bins_x * g.bins_y)

    def opts(self, **over) -> mpg_walk_opts:
        o = self.w.opts
        d = dict(max_iters=o.max_iters, tol=o.tol, beta0=o.beta0, trials=o.trials, k_max=o.k_max,
                 same_chain_eps=0.0, ray_eps=0.0, flags=o.flags, seed=o.seed, walk_id_base=o.walk_id_base,
                 max_iters_long=o.max_iters_long, recip_repeats=o.recip_repeats)
        d.update(over)
        r = mpg_walk_opts()
        for k, v in d.items():
            setattr(r, k, v)
        return r

    def close(self):
        if getattr(self, "guide", None):
            mpg_guide_destroy(self.guide)
            self.guide = None
        if getattr(self, "h", None):
            mpg_scene_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Batch:
    """Device buffers for n_recv receivers x spp walks (query, seeds, outputs)."""

    def __init__(self, xD, nD, spp: int, k: int, device="cuda"):
        import torch
        self.n_recv = int(xD.shape[0])
        self.spp = int(spp)
        self.n = self.n_recv * self.spp
        self.k = k
        f4 = lambda a: torch.cat([torch.as_tensor(np.asarray(a, np.float32)),
                                  torch.zeros(a.shape[0], 1)], 1).contiguous()
        self.xD_host = f4(xD).pin_memory() if torch.cuda.is_available() else f4(xD)
        self.nD_host = f4(nD).pin_memory() if torch.cuda.is_available() else f4(nD)
        self.xD = self.xD_host.to(device)
        self.nD = self.nD_host.to(device)
        n = max(1, self.n)
        self.xL = torch.empty(n, 4, device=device)
        self.target = torch.empty(n, 4, device=device)
        self.bin = torch.empty(n, dtype=torch.int32, device=device)
        self.chain = torch.empty(k, n, 4, device=device)
        self.status = torch.empty(n, dtype=torch.uint8, device=device)
        self.iters = torch.empty(n, dtype=torch.int16, device=device)
        self.G = torch.empty(n, device=device)
        self.T = torch.empty(n, device=device)
        self.w = torch.empty(n, device=device)
        self.trials = torch.empty(n, dtype=torch.int32, device=device)
        self.ctype_seed = torch.empty(n, dtype=torch.int32, device=device)
        self.pn = torch.empty(n, dtype=torch.float32, device=device)
        self.ctype = torch.empty(n, dtype=torch.int16, device=device)
        self.mean = torch.empty(max(1, self.n_recv), device=device)
        self.var = torch.empty(max(1, self.n_recv), device=device)
        self.stats = torch.zeros(len(STATS_FIELDS) + 8, dtype=torch.int64, device=device)
        smp = mpg_sampler_desc(0, 0, k, 0)
        self.workspace = torch.zeros(mpg_walk_workspace_size(self.n, smp, mpg_walk_opts()), dtype=torch.uint8,
                                     device=device)
        self.query = mpg_query(self.xD.data_ptr(), self.nD.data_ptr(), self.n_recv, self.spp)
        self.seeds = mpg_seed_buf(self.xL.data_ptr(), self.target.data_ptr(), self.bin.data_ptr(),
                                  self.ctype_seed.data_ptr(), self.pn.data_ptr())
        self.out = mpg_walk_buf(self.chain.data_ptr(), self.status.data_ptr(), self.iters.data_ptr(),
                                self.G.data_ptr(), self.T.data_ptr(), self.w.data_ptr(), self.trials.data_ptr(),
                                self.ctype.data_ptr())

    def stats_dict(self):
        v = self.stats.cpu().numpy().astype(np.int64)
        d = {f: int(v[i]) for i, f in enumerate(STATS_FIELDS)}
        d["by_status"] = [int(x) for x in v[len(STATS_FIELDS):]]
        return d

    def results(self):
        """Host copies of the per-walk outputs (numpy)."""
        chain = self.chain.cpu().numpy()
        return dict(pos=np.ascontiguousarray(chain[:, :, :3].transpose(1, 0, 2)),
                    prim=np.ascontiguousarray(chain[:, :, 3].view(np.int32).T),
                    status=self.status.cpu().numpy(), iters=self.iters.cpu().numpy().astype(np.int32),
                    G=self.G.cpu().numpy(), T=self.T.cpu().numpy(), w=self.w.cpu().numpy(),
                    trials=self.trials.cpu().numpy().astype(np.int64), xL=self.xL.cpu().numpy(),
                    target=self.target.cpu().numpy(), bin=self.bin.cpu().numpy(),
                    ctype=self.ctype.cpu().numpy().astype(np.int64) & 0xffff,
                    seed_ctype=self.ctype_seed.cpu().numpy().astype(np.int64), pn=self.pn.cpu().numpy())


def run_progressive(ds: DeviceScene, b: Batch, opts: mpg_walk_opts, iterations: int = 8, stream=None,
                    on_iteration=None, exchange=None, id_stride=None, reset=True):
    """configs[4] (R22): guide reset (learned branch absent) at iteration 0, then per
    iteration: seeds -> walk (+trials) -> estimator -> accumulate [-> exchange] ->
    rebuild tables from this iteration only (P:426 footnote).  Iteration it
    uses walk_id_base = base + it*id_stride (default b.n) so every iteration draws
    fresh random numbers.  `exchange(ds)` (multi-process runs, dist.exchange_guide)
    replaces this rank's histogram by the sum over ranks before the rebuild.
    reset=False keeps the caller's initial guide (e.g. photon_init)."""
    if reset:
        mpg_guide_reset(ds.guide, stream)
    base = opts.walk_id_base
    stride = b.n if id_stride is None else id_stride
    for it in range(iterations):
        opts.walk_id_base = base + it * stride
        run_step(ds, b, opts, stream, estimate=True, accumulate=True)
        if on_iteration is not None:
            on_iteration(it)
        if exchange is not None:
            exchange(ds)
        mpg_guide_rebuild(ds.guide, stream)
    opts.walk_id_base = base


def run_step(ds: DeviceScene, b: Batch, opts: mpg_walk_opts, stream=None, estimate=True, accumulate=False):
    """One pass of the hot path: seeds -> walk (+trials) -> estimator [-> guide accumulate]."""
    mpg_sample_seeds(ds.h, ds.guide, ds.sampler, b.query, opts, b.seeds, stream)
    mpg_manifold_walk(ds.h, ds.guide, ds.sampler, b.query, b.seeds, opts, b.out, b.stats, b.workspace, stream)
    if estimate:
        mpg_estimate(b.w, b.n_recv, b.spp, b.mean, b.var, stream)
    if accumulate and ds.guide is not None:
        if ds.stree:
            mpg_guide_record_samples(ds.guide, b.query, b.seeds, b.out, b.n, stream)
        else:
            mpg_guide_accumulate(ds.guide, b.query, b.out, b.n, stream)


def training_schedule(budget_passes: int, train_frac: float = 0.3):
    """The paper's online training schedule (reading R34), in passes of one walk
    per receiver: training iterations of 1, 2, 4, ... passes (doubling, Mueller 17); after an
    iteration, a new (doubled) one starts only while less than half of the training budget
    floor(train_frac * budget) is used, otherwise the current iteration continues until the
    training budget is used up; training stops at that budget.  Returns (passes per training
    iteration, render passes).  The schedule is computed by the library (mpg_training_schedule)."""
    buf = (C.c_int64 * 64)()
    n = C.c_int32()
    r = C.c_int64()
    _check(lib().mpg_training_schedule(int(budget_passes), float(train_frac), buf, 64, C.byref(n), C.byref(r)),
           "mpg_training_schedule")
    return [int(buf[i]) for i in range(n.value)], int(r.value)


def run_train_render(ds: DeviceScene, b: Batch, opts: mpg_walk_opts, budget_passes: int, stream=None,
                     photons=None, on_iteration=None, train_frac: float = 0.3):
    """Progressive train/render loop at walk level: training
    iterations by training_schedule (each guide fitted from the last iteration's samples
    only), then render passes with the final guide, splatted into a per-receiver fp64
    sum; training samples are never splatted.  photons = (n, plane_point, plane_normal)
    starts an STree guide from photons.  Returns (image, per-receiver
    variance of the pass means, schedule)."""
    import torch
    iters, render = training_schedule(budget_passes, train_frac)
    if ds.stree and iters:
        need = max(max(iters) * b.n, photons[0] if photons else 0)
        if need > ds.stree_desc.max_samples:
            raise MPGError(f"STree guide holds {ds.stree_desc.max_samples} records; this schedule needs {need} "
                           f"(DeviceScene(..., stree_capacity={need}))")
    mpg_guide_reset(ds.guide, stream)
    if photons is not None and ds.stree:
        photon_init(ds, photons[0], photons[1], photons[2], stream=stream)
    base = opts.walk_id_base
    p = 0
    for it, n_pass in enumerate(iters):
        for _ in range(n_pass):
            opts.walk_id_base = base + p * b.n
            run_step(ds, b, opts, stream, estimate=False, accumulate=True)
            p += 1
        mpg_guide_rebuild(ds.guide, stream)
        if on_iteration is not None:
            on_iteration(it, n_pass)
    dev = b.w.device
    s = torch.zeros(b.n_recv, dtype=torch.float64, device=dev)
    s2 = torch.zeros(b.n_recv, dtype=torch.float64, device=dev)
    for _ in range(render):
        opts.walk_id_base = base + p * b.n
        run_step(ds, b, opts, stream, estimate=False, accumulate=False)
        mpg_splat(b.w, b.n_recv, b.spp, s, s2, stream)
        p += 1
    opts.walk_id_base = base
    n = max(render, 1)
    img = s / n
    var = (s2 / n - img * img) * n / max(n - 1, 1)
    return img, var, (iters, render)
