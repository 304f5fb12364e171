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
print(f"cfg{cfg}: {t[0]:.2f} ms")
tr_cyc = p[2] + p[3]
print(f" trace: rounds {p[0]:,} lanes/round {p[1] / max(p[0], 1):.1f} busy {100 * p[2] / max(tr_cyc, 1):.1f}% idle rounds {p[4]:,}"
      f" cycles/round {p[2] / max(p[0], 1):.0f}")
cc = p[7] + p[10] + p[12] + p[13]
print(f" compute: solve {100 * p[7] / cc:.1f}% ({p[5]:,} batches, {p[6] / max(p[5], 1):.1f} slots, {p[7] / max(p[5], 1):.0f} cyc)"
      f" ctl {100 * p[10] / cc:.1f}% ({p[8]:,} batches, {p[9] / max(p[8], 1):.1f} slots, {p[10] / max(p[8], 1):.0f} cyc)"
      f" wait {100 * p[12] / cc:.1f}% ({p[11]:,}) idle {100 * p[13] / cc:.1f}% ({p[14]:,})")
