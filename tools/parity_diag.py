"""Diagnose GPU-vs-oracle walk disagreements (run on the GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_12818_b200 import workloads as W
from tests import parity as PY

which = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
w = {"cfg0": lambda: W.config0(), "cfg1": lambda: W.config1(128, 1), "cfg1a": lambda: W.config1(96, 2, analytic=True),
     "cfg2": lambda: W.config2(64, 4), "cfg3": lambda: W.config3(48, 1), "cfg3_64": lambda: W.config3(64, 1)}[which]()
flags = int(sys.argv[2]) if len(sys.argv) > 2 else w.opts.flags
g, st, ext = PY.run_gpu(w, flags=flags)
ids = np.arange(w.n_walks)
o, s = PY.run_oracle(w, ids)
rep = PY.compare(g, o, ids, ext, w.seed.k)
print({k: v for k, v in rep.items() if not isinstance(v, np.ndarray)})
d = rep["disagree_ids"]
tab = {}
for i in d:
    key = (int(g["status"][i]), int(o["status"][i]))
    tab[key] = tab.get(key, 0) + 1
print("disagreements (gpu_status, oracle_status):", tab)
print("gpu iters:", g["iters"][d][:40])
print("orc iters:", o["iters"][d][:40])
# both converged, different chains
both = np.isin(g["status"], (0, 5)) & np.isin(o["status"], (0, 5))
dp = np.linalg.norm(g["pos"][:, :w.seed.k] - o["pos"][:, :w.seed.k], axis=2).max(1) / ext
far = np.nonzero(both & (dp > 1e-4))[0]
print("both converged but different chain:", len(far), dp[far][:10])
print("iteration histogram (oracle converged):", np.bincount(o["iters"][np.isin(o["status"], (0, 5))], minlength=21))
# boundary classification (reading R18): oracle outcome under 8 seed perturbations of 1e-4*extent
rng = np.random.default_rng(0)
nb = 0
for i in d[:200]:
    tgt = o["target"][i].astype(np.float64)
    xD = w.xD[i // w.spp].astype(np.float64)
    base = np.isin(o["status"][i], (0, 5))
    changed = False
    for j in range(8):
        v = rng.normal(size=3); v /= np.linalg.norm(v)
        r = s.walk_from_target(xD, w.nD[0], o["xL"][i], tgt + 1e-4 * ext * v)
        if (r["status"] in (0, 5)) != base:
            changed = True
            break
    nb += changed
print(f"boundary (seed perturbation): {nb} of {min(200, len(d))} disagreements")
# iteration-budget boundary: the oracle's flag changes with max_iters in [max-3, max+3]
nbi = 0
for i in d[:200]:
    xD = w.xD[i // w.spp].astype(np.float64)
    base = np.isin(o["status"][i], (0, 5))
    fl = []
    for mi in (w.opts.max_iters - 3, w.opts.max_iters + 3):
        r = s.walk_from_target(xD, w.nD[0], o["xL"][i], o["target"][i].astype(np.float64), opts=s.opts(max_iters=mi))
        fl.append(r["status"] in (0, 5))
    nbi += (fl[0] != base) or (fl[1] != base)
print(f"boundary (iteration budget +-3): {nbi} of {min(200, len(d))} disagreements")

# per-iteration traces of a few disagreements: GPU vs oracle
import torch
from paper_2311_12818_b200 import mpg
ds = mpg.DeviceScene(w)
b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
stride = 2 * (w.opts.max_iters + 2)
buf = torch.full((w.n_walks, stride), -1.0, device="cuda")
mpg.mpg_debug_trace(buf, w.n_walks, stride)
mpg.run_step(ds, b, ds.opts(flags=flags))
torch.cuda.synchronize()
mpg.mpg_debug_trace(None)
tr = buf.cpu().numpy()
st2 = b.status.cpu().numpy(); it2 = b.iters.cpu().numpy()
print("rerun determinism: status equal", (st2 == g["status"]).mean(), "iters equal", (it2 == g["iters"]).mean())
np.set_printoptions(precision=3, linewidth=250)
for i in d[:8]:
    st_o, it_o, res_o, beta_o = s.walk_trace(w.xD[i // w.spp].astype(np.float64), o["xL"][i], o["target"][i].astype(np.float64))
    ng = g["iters"][i] + 1
    print(f"walk {i}: gpu status {g['status'][i]} it {g['iters'][i]}; oracle {st_o} it {it_o}")
    print("  gpu res :", tr[i, 0:2 * ng:2])
    print("  orc res :", res_o)
    print("  gpu beta:", tr[i, 1:2 * ng:2])
    print("  orc beta:", beta_o)
