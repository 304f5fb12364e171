"""Glossy separator (Eq. 14; R35) on configs[4]: the STree guide fitted with the
product weighting rho(w_v, w_D*) w vs with w alone, then render passes whose estimate is
rho * w (the separator's BSDF times the walk weight).  Reports the variance of that image at
equal budget.  rho for the measurement is evaluated here with torch (tool-side only).
Usage (GPU box): python tools/glossy_compare.py [alpha] [train_iters] [render_passes]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_12818_b200 import mpg, workloads as W  # noqa: E402


def rho(n, wv, om, alpha):
    cv = (n * wv).sum(1)
    cl = (n * om).sum(1)
    h = wv + om
    h = h / h.norm(dim=1, keepdim=True)
    nh = (n * h).sum(1)
    a2 = alpha * alpha
    t = nh * nh * (a2 - 1) + 1
    D = a2 / (np.pi * t * t)
    r = D / (4 * cv * cl)
    return torch.where((cv > 0) & (cl > 0), r, torch.zeros_like(r))


def main():
    alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    passes = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    w = W.config4(guide="stree")
    eye = np.array([2.0, 6.0, -4.0])
    wv = eye[None, :] - w.xD.astype(np.float64)
    wv = wv / np.linalg.norm(wv, axis=1, keepdims=True)
    wv4 = torch.zeros(len(wv), 4, device="cuda")
    wv4[:, :3] = torch.from_numpy(wv).float().cuda()
    out = {"alpha": alpha, "train_iterations": iters, "render_passes": passes, "rows": []}
    for product in (False, True):
        ds = mpg.DeviceScene(w)
        b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
        opts = ds.opts(flags=w.opts.flags | 8)
        if product:
            mpg.mpg_guide_set_separator(ds.guide, wv4, b.nD, alpha)
        mpg.mpg_guide_reset(ds.guide)
        p = 0
        for it in range(iters):
            opts.walk_id_base = p * b.n
            mpg.run_step(ds, b, opts, accumulate=True)
            mpg.mpg_guide_rebuild(ds.guide)
            p += 1
        s = torch.zeros(b.n_recv, dtype=torch.float64, device="cuda")
        s2 = torch.zeros_like(s)
        n3 = b.nD[:, :3]
        for _ in range(passes):
            opts.walk_id_base = p * b.n
            mpg.run_step(ds, b, opts)
            om = b.chain[0, :, :3] - b.xD[:, :3]
            om = om / om.norm(dim=1, keepdim=True).clamp_min(1e-30)
            e = (rho(n3, wv4[:, :3], om, alpha) * b.w).double()
            e = torch.nan_to_num(e)
            s += e
            s2 += e * e
            p += 1
        torch.cuda.synchronize()
        img = s / passes
        var = (s2 / passes - img * img) * passes / (passes - 1) / passes
        row = dict(product_weighting=product, image_mean=float(img.mean()), image_variance=float(var.mean()),
                   p99_pixel_variance=float(torch.quantile(var.float(), 0.99)))
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
        ds.close()
    out["variance_ratio_product_over_plain"] = out["rows"][1]["image_variance"] / out["rows"][0]["image_variance"]
    print(json.dumps(out), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "glossy_compare.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
