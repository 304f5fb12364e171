"""k_walk activity over time (diagnostic build, run on the GPU box).

    python tools/timeline.py [config] [bin_ms]

Builds libmpg_tl.so with -DMPG_TIMELINE (one ballot + 4 atomics per warp
iteration), runs the bench step of a config a few times and prints, per time
bin: warp iterations, mean lanes tracing / working / waiting per iteration.
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TL = os.path.join(ROOT, "paper_2311_12818_b200", "libmpg_tl.so")
if not os.path.exists(TL):
    from paper_2311_12818_b200 import build as B
    subprocess.check_call([B.NVCC] + B.FLAGS + ["-DMPG_TIMELINE", "-o", TL, B.SRC])
os.environ["MPG_LIB"] = TL

import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2311_12818_b200 import mpg, workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
bin_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
shift = int(sys.argv[3]) if len(sys.argv) > 3 else 16      # bucket = 2^shift ns (1024 buckets)
w = W.CONFIGS[cfg]()
ds = mpg.DeviceScene(w)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
opts = ds.opts(flags=w.opts.flags | 8)   # bench default: MPG_FLAG_SORT
L = mpg.lib()
fn = C.CDLL(TL).mpg_debug_timeline
buf = (C.c_ulonglong * 6144)()
nh = (C.c_ulonglong * 256)()
for rep in range(3):
    mpg.mpg_sample_seeds(ds.h, ds.guide, ds.sampler, b.query, opts, b.seeds)
    torch.cuda.synchronize()
    fn(buf, shift, nh)   # zero
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mpg.mpg_manifold_walk(ds.h, ds.guide, ds.sampler, b.query, b.seeds, opts, b.out, b.stats, b.workspace)
    e1.record()
    torch.cuda.synchronize()
    fn(buf, shift, nh)
    ms = e0.elapsed_time(e1)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 6).astype(np.float64)
nz = np.nonzero(a[:, 0])[0]
# buckets wrap every 1024 x 2^shift ns: start after the largest empty gap
gaps = np.diff(np.r_[nz, nz[0] + 1024])
s = nz[(np.argmax(gaps) + 1) % len(nz)]
seq = [(s + i) % 1024 for i in range(1024)]
rows = a[seq]
last = np.nonzero(rows[:, 0])[0].max()
rows = rows[:last + 1]
bw = 2.0 ** shift / 1e6   # ms per bucket
per = max(1, int(round(bin_ms / bw)))
print(f"config {cfg}: k_walk {ms:.2f} ms, {rows[:, 0].sum():.0f} warp iterations, "
      f"trace lanes/iter {rows[:, 1].sum() / rows[:, 0].sum():.2f}")
print("   t_ms iters(M)  tracing  working  waiting  primary    items")
for i in range(0, len(rows), per):
    r = rows[i:i + per].sum(0)
    if r[0] == 0:
        continue
    print(f"{i * bw:7.2f} {r[0] / 1e6:8.3f} " + " ".join(f"{r[j] / r[0]:8.2f}" for j in range(1, 6)))
h = np.frombuffer(nh, dtype=np.uint64).astype(np.float64)
if h.sum():
    c = np.cumsum(h) / h.sum()
    mean = (h * np.arange(256)).sum() / h.sum()
    q = {p: int(np.searchsorted(c, p)) for p in (0.5, 0.9, 0.99, 0.999)}
    # expected max over 32 i.i.d. lanes: sum over v of 1 - F(v)^32
    emax = float(np.sum(1.0 - c[:-1] ** 32))
    print(f"closest-hit rays: {h.sum():.0f}, node visits mean {mean:.1f}, quantiles {q}, E[max of 32] {emax:.1f}")
ds.close()
