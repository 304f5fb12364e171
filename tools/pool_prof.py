"""Role utilisation of the pool kernel (MPG_POOL_PROF build): python tools/pool_prof.py cfg [env knobs]"""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_12818_b200 import mpg
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import pool_check as PC

cfg = int(sys.argv[1])
small = "--small" in sys.argv
w = PC.make(cfg, small)
ds = mpg.DeviceScene(w)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
fl = w.opts.flags | 8 | (4 if cfg >= 1 else 0)
opts = ds.opts(flags=fl)
L = mpg.lib()
out = (C.c_ulonglong * 16)()
r, s, t = PC.run(ds, b, opts, 1, 2)
L.mpg_debug_pool_prof(out)
r, s, t = PC.run(ds, b, opts, 1, 1)
L.mpg_debug_pool_prof(out)
p = [int(x) for x in out]
print(f"cfg{cfg}: {t[0]:.2f} ms  env " + " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("MPG_POOL")))
tot = p[2] + p[3] + p[7] + p[10] + p[11]
nw = 148 * int(os.environ.get("NW", "20"))
print(f" warp-cycles: R {100 * p[2] / tot:.1f}% H {100 * p[3] / tot:.1f}% S {100 * p[7] / tot:.1f}% C {100 * p[10] / tot:.1f}% scheduler+barriers {100 * p[11] / tot:.1f}%")
print(f" phases per block: R {p[0] / nw:.0f} H {p[12] / nw:.0f} S {p[1] / nw:.0f} C {p[4] / nw:.0f}; cycles per phase: R {p[2] / max(p[0], 1):.0f} H {p[3] / max(p[12], 1):.0f} S {p[7] / max(p[1], 1):.0f} C {p[10] / max(p[4], 1):.0f};"
      f" solve batches {p[5]:,} x {p[6] / max(p[5], 1):.1f} slots; control batches {p[8]:,} x {p[9] / max(p[8], 1):.1f} slots")
