"""Time mpg_manifold_walk under trial-schedule knobs (env, read at every launch).

    python tools/tail_sweep.py <config> "B0,GROW,LOCAL,BACKOFF,GROW_IDLE,IDLE_DIV,B0_IDLE" ...

Each setting: MPG_ITEM_B0 (first item batch), MPG_ITEM_GROW (batch shift),
MPG_LOCAL_TRIALS (sequential trials before a walk becomes a hard entry),
MPG_BACKOFF_MAX (ns); '-' keeps the library default.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_12818_b200 import mpg, workloads as W  # noqa: E402

cfg = int(sys.argv[1])
settings = sys.argv[2:] or ["-,-,-,-"]
w = W.CONFIGS[cfg]()
ds = mpg.DeviceScene(w)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
opts = ds.opts(flags=w.opts.flags | 8)
mpg.mpg_sample_seeds(ds.h, ds.guide, ds.sampler, b.query, opts, b.seeds)
names = ["MPG_ITEM_B0", "MPG_ITEM_GROW", "MPG_LOCAL_TRIALS", "MPG_BACKOFF_MAX", "MPG_ITEM_GROW_IDLE", "MPG_IDLE_DIV", "MPG_ITEM_B0_IDLE"]
ref = None
for s in settings:
    for n, v in zip(names, s.split(",")):
        if v == "-":
            os.environ.pop(n, None)
        else:
            os.environ[n] = v
    ts = []
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mpg.mpg_manifold_walk(ds.h, ds.guide, ds.sampler, b.query, b.seeds, opts, b.out, b.stats, b.workspace)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = b.stats_dict()
    print(f"cfg{cfg} {s:>24s}: {sorted(ts[1:])[1]:8.2f} ms (min {min(ts[1:]):.2f})  attempts={st['attempts']} "
          f"trials={st['trials']} trunc={st['truncated']}", flush=True)
ds.close()
