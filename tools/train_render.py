"""configs[4] at full size: the progressive train/render loop at equal
budget -- untrained render vs the paper's schedule with the histogram guide, the STree
guide and the photon-started STree guide.  Reports the variance of the final image
(mean over receivers of the pass variance / render passes), the time, and the
efficiency 1 / (variance x time).  Usage (GPU box): python tools/train_render.py [budget]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2311_12818_b200 import mpg, workloads as W  # noqa: E402


def main():
    budget = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    rows = []
    runs = [("untrained", "hist", 0.0, None, 300.0), ("hist", "hist", 0.3, None, 300.0),
            ("stree", "stree", 0.3, None, 300.0),
            ("stree+photons", "stree", 0.3, (1 << 20, (0, -2, 0), (0, 1, 0)), 300.0)]
    if len(sys.argv) > 2:   # kappa_max sweep of the STree guide (R30 clamp)
        runs = [(f"stree kappa_max={k}", "stree", 0.3, None, float(k)) for k in sys.argv[2].split(",")]
    for name, guide, frac, photons, kmax in runs:
        w = W.config4(guide=guide)
        iters, _ = mpg.training_schedule(budget, frac)
        ds = mpg.DeviceScene(w, stree_capacity=max([1] + iters) * w.n_walks, stree_kappa=(1.0 if kmax < 3e38 else 0.0, kmax))
        b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
        opts = ds.opts(flags=w.opts.flags | 8)
        mpg.run_train_render(ds, b, opts, 4, train_frac=frac, photons=photons)     # warm-up (allocations)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        img, var, sched = mpg.run_train_render(ds, b, opts, budget, train_frac=frac, photons=photons)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        v_img = float(var.mean()) / max(sched[1], 1)
        vr = var / max(sched[1], 1)
        row = dict(run=name, schedule=sched, ms=ms, image_mean=float(img.mean()), image_variance=v_img,
                   efficiency=1.0 / (v_img * ms), median_pixel_variance=float(vr.median()),
                   p99_pixel_variance=float(torch.quantile(vr.float(), 0.99)), max_pixel_variance=float(vr.max()))
        rows.append(row)
        print(json.dumps(row), flush=True)
        ds.close()
    for r in rows:
        r["efficiency_vs_untrained"] = r["efficiency"] / rows[0]["efficiency"]
        r["variance_vs_untrained"] = r["image_variance"] / rows[0]["image_variance"]
    out = {"budget_passes": budget, "walks_per_pass": 1 << 20, "rows": rows}
    print(json.dumps(out), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = "_kappa" if len(sys.argv) > 2 else ""
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"train_render_{budget}{tag}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
