"""CPU checks of the C ABI boundary: the library loads, exports every symbol
include/mpg.h declares, and rejects bad arguments synchronously (no GPU needed)."""
import ctypes as C
import os
import re

import pytest

from paper_2311_12818_b200 import mpg, build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    return mpg.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mpg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["mpg_scene_create", "mpg_guide_upload", "mpg_sample_seeds", "mpg_manifold_walk",
              "mpg_guide_accumulate"]:
        assert s in syms


def test_library_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert set(syms) == set(mpg.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s


def test_version(L):
    assert mpg.mpg_version() == 1


def test_invalid_arguments_rejected_synchronously(L):
    h = C.c_void_p()
    assert L.mpg_scene_create(None, 0, None, 0, None, C.byref(h)) == 1
    assert b"surfaces" in L.mpg_last_error()
    g = mpg.mpg_guide_desc()
    assert L.mpg_guide_create(C.byref(g), C.byref(h)) == 1
    assert L.mpg_estimate(None, 1, 1, None, None, None) == 1
    q = mpg.mpg_query()
    sd = mpg.mpg_sampler_desc()
    o = mpg.mpg_walk_opts()
    s = mpg.mpg_seed_buf()
    wb = mpg.mpg_walk_buf()
    assert L.mpg_manifold_walk(None, None, C.byref(sd), C.byref(q), C.byref(s), C.byref(o), C.byref(wb), None,
                               None, 0, None) == 1
    assert L.mpg_walk_workspace_size(10, C.byref(sd), C.byref(o)) >= 8


def test_struct_layouts():
    # layouts mirrored by the binding (natural alignment, see include/mpg.h)
    assert C.sizeof(mpg.mpg_walk_opts) == 56
    assert C.sizeof(mpg.mpg_walk_stats) == 19 * 8
    assert C.sizeof(mpg.mpg_query) == 32
    assert C.sizeof(mpg.mpg_sampler_desc) == 16


def test_stree_photon_splat_arguments_rejected_synchronously(L):
    """The 8(f) entry points check their arguments before touching the device."""
    h = C.c_void_p()
    d = mpg.mpg_stree_desc(max_samples=10, eps=0.6, c_thr=1.0, kappa_min=1.0, kappa_max=300.0, max_depth=32)
    assert L.mpg_guide_create_stree(C.byref(d), C.byref(h)) == 1 and b"eps" in L.mpg_last_error()
    d.eps, d.kappa_min, d.kappa_max = 0.1, 5.0, 1.0
    assert L.mpg_guide_create_stree(C.byref(d), C.byref(h)) == 1 and b"kappa" in L.mpg_last_error()
    d.kappa_min, d.kappa_max, d.max_depth = 1.0, 300.0, 99
    assert L.mpg_guide_create_stree(C.byref(d), C.byref(h)) == 1
    assert L.mpg_guide_create_stree(None, C.byref(h)) == 1
    assert L.mpg_guide_set_separator(None, None, None, C.c_float(0.1)) == 1
    assert L.mpg_guide_set_samples(None, None, 0, None) == 1
    info = mpg.mpg_stree_info()
    assert L.mpg_guide_stree_info(None, C.byref(info)) == 1
    p = mpg.mpg_photon_desc(n_photons=10, max_vertices=7)
    assert L.mpg_trace_photons(None, C.byref(p), None, None) == 1
    assert L.mpg_splat(None, 1, 1, None, None, None) == 1


def test_new_struct_layouts():
    assert C.sizeof(mpg.mpg_stree_desc) == 32
    assert C.sizeof(mpg.mpg_stree_info) == 48
    assert C.sizeof(mpg.mpg_photon_desc) == 56
    assert mpg.GUIDE_SAMPLE_BYTES == 48


def test_trace_loop_head_yields_in_every_walk_kernel(L, tmp_path):
    """DESIGN.md §4 item 1: the per-ray loop of trace_chain starts with a YIELD (emitted
    because of the shared-memory ray counter in that loop), which lets lanes that are done
    with ray i go on while warp-mates still traverse (measured -7..-17 % k_walk time).
    ptxas decides this, so the built SASS is checked: every k_walk instantiation has a
    YIELD directly before the code of the trace_chain loop."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    nvdisasm = shutil.which("nvdisasm") or "/usr/local/cuda/bin/nvdisasm"
    if not (os.path.exists(cuobjdump) and os.path.exists(nvdisasm)):
        pytest.skip("CUDA binary utilities not available")
    src = open(os.path.join(ROOT, "paper_2311_12818_b200", "csrc", "walk.cuh")).read().splitlines()
    start = next(i for i, l in enumerate(src) if "int trace_chain(" in l) + 1
    end = next(i for i, l in enumerate(src) if i > start and "tau_res = res;" in l) + 1
    subprocess.run([cuobjdump, "-xelf", "all", mpg.LIB_PATH], cwd=tmp_path, check=True, capture_output=True)
    cub = [f for f in os.listdir(tmp_path) if f.endswith(".cubin")]
    assert cub
    sass = subprocess.run([nvdisasm, "-g", "-c", str(tmp_path / cub[0])], capture_output=True, text=True).stdout
    kernels, fn, cur = {}, None, None
    for line in sass.splitlines():
        if ".section\t.text." in line:
            name = line.split(".text.")[1].split(",")[0]
            fn = name if name.startswith("_Z6k_walk") else None
            if fn:
                kernels[fn] = []
            continue
        if fn is None:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        if re.search(r"/\*[0-9a-f]{4,}\*/", line):
            kernels[fn].append((cur, line))
    assert len(kernels) >= 8
    for fn, ins in kernels.items():
        m = re.search(r"ELb([01])ELb([01])EE", fn)       # k_walk<KMAX, R, W, MINB, GL, CMP>
        if m and m.group(2) == "1":
            continue                                     # compacted rounds: no per-lane ray loop
        ok = False
        for j, (c, l) in enumerate(ins):
            if "YIELD" not in l:
                continue
            nxt = [x for x, _ in ins[j + 1:j + 6] if x]
            if any(f == "walk.cuh" and start <= n <= end for f, n in nxt):
                ok = True
                break
        assert ok, f"no YIELD at the trace_chain loop head in {fn}"
