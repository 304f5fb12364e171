import sys, numpy as np
sys.path.insert(0, ".")
from paper_2311_12818_b200 import workloads as W
from tests import parity as PY
for mk in [lambda: W.config1(n_side=256, spp=2), lambda: W.config0(), lambda: W.config3(n_side=64, spp=1)]:
    w = mk()
    a, sa, _ = PY.run_gpu(w)
    b, sb, _ = PY.run_gpu(w, flags=w.opts.flags | 8)
    same = all(np.array_equal(a[k], b[k]) for k in ("status", "trials", "pos", "G"))
    print(w.name, "identical:", same, {k: int((a[k] != b[k]).sum()) for k in ("status", "trials")})
