"""Progressive train/render loop (mpg.run_train_render) on the GPU:
the splat equals the mean of the render passes' weights, the image is unbiased against
an untrained render of the same budget, and training lowers its variance."""
import numpy as np
import pytest

from paper_2311_12818_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_splat_is_the_mean_of_render_passes():
    import torch
    from paper_2311_12818_b200 import mpg
    w = W.config0(n_side=16, spp=4)
    ds = mpg.DeviceScene(w)
    b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
    opts = ds.opts()
    s = torch.zeros(b.n_recv, dtype=torch.float64, device="cuda")
    ws = []
    for p in range(3):
        opts.walk_id_base = p * b.n
        mpg.run_step(ds, b, opts, estimate=False)
        mpg.mpg_splat(b.w, b.n_recv, b.spp, s)
        torch.cuda.synchronize()
        ws.append(b.w.double().cpu().numpy().reshape(b.n_recv, b.spp).mean(1))
    ds.close()
    assert np.allclose(s.cpu().numpy(), np.sum(ws, 0), rtol=1e-12, atol=0)


@pytest.mark.parametrize("guide", ["hist", "stree"])
def test_trained_render_unbiased_and_lower_variance(guide):
    from paper_2311_12818_b200 import mpg
    w = W.config4(n_side=64, guide=guide)
    res = {}
    for frac in (0.0, 0.3):
        ds = mpg.DeviceScene(w, stree_capacity=8 * w.n_walks)
        b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
        img, var, sched = mpg.run_train_render(ds, b, ds.opts(), 24, train_frac=frac)
        res[frac] = (img.cpu().numpy(), var.cpu().numpy(), sched)
        ds.close()
    (i0, v0, s0), (i1, v1, s1) = res[0.0], res[0.3]
    print(guide, s0, s1, i0.mean(), i1.mean(), v0.mean(), v1.mean())
    assert s0 == ([], 24) and s1 == ([1, 2, 4], 17)
    # same target: the whole-image means agree within their standard errors
    se = np.sqrt(v0.sum() / s0[1] + v1.sum() / s1[1]) / len(i0)
    assert abs(i0.mean() - i1.mean()) < 4 * se
    # the trained guide lowers the per-pass variance (converged walks, fewer trials)
    assert v1.mean() < v0.mean()
