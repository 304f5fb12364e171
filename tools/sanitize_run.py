"""Small end-to-end runs for compute-sanitizer: every kernel of the walk path
on small inputs, with the trial entry table / item ring shrunk (MPG_TEST_HARD_CAP /
MPG_TEST_ITEM_CAP set by the caller) so the fallback paths run too.
usage (GPU box): compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2311_12818_b200 import mpg, workloads as W

runs = [("cfg0", W.config0(n_side=32, spp=4)), ("cfg0v", W.config0(n_side=16, spp=4, occluders=True)),
        ("cfg1", W.config1(n_side=48)), ("cfg2", W.config2(n_side=32, spp=2, grid_n=64)),
        ("cfg3", W.config3(n_side=24, grid_n=32)), ("cfg4", W.config4(n_side=48, grid_n=64))]
for name, w in runs:
    ds = mpg.DeviceScene(w)
    b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
    opts = ds.opts(flags=w.opts.flags | 8)
    if w.seed.mode == W.SEED_GUIDE_DIR:
        mpg.run_progressive(ds, b, opts, iterations=2)
    else:
        mpg.run_step(ds, b, opts, accumulate=ds.guide is not None)
    torch.cuda.synchronize()
    st = b.stats_dict()
    print(name, "walks", st["walks"], "converged", st["converged"], "trials", st["trials"], flush=True)
    ds.close()
# the STree guide: records -> rebuild -> guided walk with selective activation; photons
w = W.config4(n_side=48, grid_n=64, guide="stree")
ds = mpg.DeviceScene(w, stree_capacity=1 << 16)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
mpg.mpg_guide_reset(ds.guide)
mpg.photon_init(ds, 1 << 14, (0, -2, 0), (0, 1, 0))
mpg.run_progressive(ds, b, ds.opts(flags=w.opts.flags | 8 | 16), iterations=2, reset=False)
torch.cuda.synchronize()
print("stree", b.stats_dict()["by_status"], flush=True)
ds.close()
# R x M repetitions
w = W.config1(n_side=32)
ds = mpg.DeviceScene(w)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
mpg.run_step(ds, b, ds.opts(recip_repeats=3))
torch.cuda.synchronize()
print("rxm", b.stats_dict()["trials"], flush=True)
ds.close()
print("SANITIZE_RUN_DONE")
