"""Per-iteration ||C||_inf of chosen walks, GPU (mpg_debug_trace, fp32 copy of the fp64
residual) vs oracle (orc_walk_trace), to full float precision (run on the GPU box).
usage: python tools/trace_compare.py cfg3_64 3733 3736 ..."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2311_12818_b200 import mpg, workloads as W
from oracle import oracle as O

which = sys.argv[1]
ids = [int(a) for a in sys.argv[2:]]
w = {"cfg3_64": lambda: W.config3(64, 1), "cfg1": lambda: W.config1(128, 1)}[which]()
ds = mpg.DeviceScene(w)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
mi = max(w.opts.max_iters, w.opts.max_iters_long)
stride = 2 * (mi + 2)
buf = torch.full((w.n_walks, stride), -1.0, device="cuda")
mpg.mpg_debug_trace(buf, w.n_walks, stride)
mpg.run_step(ds, b, ds.opts(trials=0))
torch.cuda.synchronize()
mpg.mpg_debug_trace(None)
tr = buf.cpu().numpy()
g = b.results()
s = O.OracleScene(w)
o = s.walks(np.asarray(ids), s.opts(trials=0))
for j, i in enumerate(ids):
    st, it, res, beta = s.walk_trace(w.xD[i // w.spp].astype(np.float64), o["xL"][j], o["target"][j].astype(np.float64))
    print(f"walk {i}: gpu status {g['status'][i]} it {g['iters'][i]}  oracle {st} it {it}")
    gi = 0
    for k in range(min(int(g["iters"][i]), it) + 1):
        gr, gb = tr[i, 2 * k], tr[i, 2 * k + 1]
        orr = res[k] if k < len(res) else float("nan")
        ob = beta[k] if k < len(beta) else float("nan")
        rel = abs(gr - orr) / max(abs(orr), 1e-30) if gr >= 0 else float("nan")
        print(f"  it {k:2d}  gpu {gr: .7e} b={gb:.6f}   orc {orr: .7e} b={ob:.6f}   rel {rel:.1e}")
