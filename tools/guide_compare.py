"""Histogram guide vs the paper's STree + vMF guide on configs[4] at equal walk budget
("compare variance against the histogram at equal walk budget").

Runs the progressive loop (guide reset, 8 iterations x n walks, each iteration's
guide fitted from the previous iteration's samples) with each guide and reports,
per iteration: converged walks, the estimator mean E[w] over all walks (both
guides are unbiased for the same sum of throughputs, Eq. 3), the second moment
E[w^2] and the variance of w (lower = better guide), the rebuild time, and for
the STree its size.  Usage (GPU box):  python tools/guide_compare.py [n_side] [iters]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_12818_b200 import mpg, workloads as W  # noqa: E402


def run(guide, n_side, iters):
    photons = guide.endswith("+photons")          # photon-based p_0
    w = W.config4(n_side=n_side, guide=guide.split("+")[0])
    ds = mpg.DeviceScene(w, stree_capacity=max(n_side * n_side, 1 << 20))
    b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
    opts = ds.opts(flags=w.opts.flags | 8)
    rows = []
    mpg.mpg_guide_reset(ds.guide)
    if photons:
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        landed = mpg.photon_init(ds, 1 << 20, (0, -2, 0), (0, 1, 0), seed=1)
        e[1].record()
        torch.cuda.synchronize()
        print(guide, json.dumps({"photons": 1 << 20, "landed": landed, "ms": e[0].elapsed_time(e[1]),
                                 "tree": mpg.mpg_guide_stree_info(ds.guide)}), flush=True)
    for it in range(iters):
        opts.walk_id_base = it * b.n
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        mpg.run_step(ds, b, opts, accumulate=True)
        e[1].record()
        mpg.mpg_guide_rebuild(ds.guide)
        e[2].record()
        torch.cuda.synchronize()
        wv = b.w.double()
        st = b.stats_dict()
        row = dict(it=it, converged=st["converged"], mean_w=float(wv.mean()), second_moment=float((wv * wv).mean()),
                   var_w=float(wv.var()), step_ms=e[0].elapsed_time(e[1]), rebuild_ms=e[1].elapsed_time(e[2]),
                   trials_per_conv=st["trials"] / max(1, st["converged"]), newton_iters=st["newton_iters"])
        if guide.startswith("stree"):
            row["tree"] = mpg.mpg_guide_stree_info(ds.guide)
        rows.append(row)
        print(guide, json.dumps(row), flush=True)
    ds.close()
    return rows


os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)


def main():
    n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    out = {"n_side": n_side, "walks_per_iteration": n_side * n_side, "iterations": iters}
    guides = sys.argv[3].split(",") if len(sys.argv) > 3 else ["hist", "stree"]
    for g in guides:
        t0 = time.time()
        out[g] = run(g, n_side, iters)
        out[g + "_wall_s"] = time.time() - t0
    if "hist" not in guides or "stree" not in guides:
        json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"guide_compare_{n_side}_{'_'.join(guides)}.json"), "w"),
                  indent=1)
        return
    last = {g: out[g][-1] for g in ("hist", "stree")}
    out["summary"] = {
        "mean_w": {g: last[g]["mean_w"] for g in last},
        "var_w_last_iteration": {g: last[g]["var_w"] for g in last},
        "variance_ratio_stree_over_hist": last["stree"]["var_w"] / max(last["hist"]["var_w"], 1e-300),
        "converged_last_iteration": {g: last[g]["converged"] for g in last},
        "mean_rebuild_ms": {g: float(np.mean([r["rebuild_ms"] for r in out[g][1:]])) for g in last},
    }
    print(json.dumps(out["summary"]), flush=True)
    for g in guides:
        if g not in ("hist", "stree"):
            out["summary"]["converged_per_iteration_" + g] = [r["converged"] for r in out[g]]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"guide_compare_{n_side}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
