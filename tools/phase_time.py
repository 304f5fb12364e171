"""Time mpg_manifold_walk alone (CUDA events) for a config with trials on/off and
several k_max: separates the primary phase from the trial tail (MPG_LIB override)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2311_12818_b200 import mpg, workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = W.CONFIGS[cfg]()
ds = mpg.DeviceScene(w)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
for trials, kmax in [(0, 1), (1, 4), (1, 8), (1, 32), (1, 128), (1, 1024)]:
    opts = ds.opts(trials=trials, k_max=kmax, flags=w.opts.flags | 8)
    mpg.mpg_sample_seeds(ds.h, ds.guide, ds.sampler, b.query, opts, b.seeds)
    ts = []
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mpg.mpg_manifold_walk(ds.h, ds.guide, ds.sampler, b.query, b.seeds, opts, b.out, b.stats, b.workspace)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = b.stats_dict()
    print(f"cfg{cfg} trials={trials} k_max={kmax:5d}: {min(ts[1:]):8.2f} ms  attempts={st['attempts']} trials={st['trials']}")
ds.close()
