"""Compare per-walk trial counts of two builds (MPG_LIB override) on configs[0]."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, ".")
code = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_2311_12818_b200 import workloads as W
from tests import parity as PY
w = W.config0()
g, st, ext = PY.run_gpu(w)
np.savez(sys.argv[1], trials=g["trials"], status=g["status"], w=g["w"], T=g["T"])
print(json.dumps({"stats_trials": st["trials"], "sum": int(g["trials"].astype(np.int64).sum()), "trunc": st["truncated"]}))
'''
res = {}
for lib in sys.argv[1:]:
    env = dict(os.environ, MPG_LIB=lib)
    out = subprocess.run([sys.executable, "-c", code, f"/tmp/{os.path.basename(lib)}.npz"], env=env,
                         capture_output=True, text=True)
    print(lib, out.stdout.strip()[-300:], out.stderr.strip()[-300:])
    res[lib] = np.load(f"/tmp/{os.path.basename(lib)}.npz")
a, b = [res[l] for l in sys.argv[1:3]]
d = np.nonzero(a["trials"] != b["trials"])[0]
print("walks with different trials:", len(d))
for i in d[:20]:
    print(i, a["status"][i], b["status"][i], a["trials"][i], b["trials"][i], a["w"][i], b["w"][i])
