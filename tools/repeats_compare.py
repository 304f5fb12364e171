"""R x M: per-pixel variance and cost of averaging M reciprocal-probability
estimates, at full size on configs[1] (or another config).  Two independent runs
(walk_id_base 0 and n) give the per-pixel variance of the estimate as
mean((w_a - w_b)^2) / 2; efficiency = 1 / (variance x time).
Usage (GPU box): python tools/repeats_compare.py [config] [M list, e.g. 1,2,4]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_12818_b200 import mpg, workloads as W  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    Ms = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4").split(",")]
    w = W.CONFIGS[cfg]()
    ds = mpg.DeviceScene(w)
    b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
    rows = []
    for M in Ms:
        runs, ms = [], []
        for rep in range(3):
            opts = ds.opts(flags=w.opts.flags | 8, recip_repeats=M, walk_id_base=(rep % 2) * b.n)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mpg.run_step(ds, b, opts)
            e1.record()
            torch.cuda.synchronize()
            if rep > 0:
                ms.append(e0.elapsed_time(e1))
            runs.append(b.mean[:b.n_recv].double().cpu().numpy())
        a, c = runs[1], runs[2]          # walk_id_base n and 0: independent draws
        var = float(np.mean((a - c) ** 2) / 2.0)
        t = float(np.mean(ms))
        st = b.stats_dict()
        row = dict(M=M, ms_per_step=t, pixel_variance=var, mean_estimate=float((a.mean() + c.mean()) / 2),
                   efficiency=1.0 / (var * t), trials_per_step=st["trials"], attempts=st["attempts"])
        rows.append(row)
        print(json.dumps(row), flush=True)
    base = rows[0]
    for r in rows:
        r["variance_ratio"] = r["pixel_variance"] / base["pixel_variance"]
        r["time_ratio"] = r["ms_per_step"] / base["ms_per_step"]
        r["efficiency_ratio"] = r["efficiency"] / base["efficiency"]
    out = {"config": cfg, "n_walks": b.n, "rows": rows}
    print(json.dumps(out), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"repeats_cfg{cfg}.json"), "w"), indent=1)
    ds.close()


if __name__ == "__main__":
    main()
