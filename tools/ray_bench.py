"""Ray-engine microbenchmark: mpg_trace_rays (one ray per thread) on ray
batches shaped like a walk's rays, to size the traversal ceiling.

usage (GPU box): python tools/ray_bench.py [config] [n_rays]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_12818_b200 import mpg, workloads as W  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 23
    w = W.CONFIGS[cfg]()
    ds = mpg.DeviceScene(w)
    g = torch.Generator(device="cuda").manual_seed(0)
    P = torch.tensor(np.concatenate([s.positions for s in w.surfaces if s.positions is not None]),
                     device="cuda", dtype=torch.float32)
    xD = torch.as_tensor(w.xD, device="cuda")[:, :3]
    ri = torch.randint(0, xD.shape[0], (n,), device="cuda", generator=g)
    vi = torch.randint(0, P.shape[0], (n,), device="cuda", generator=g)
    vj = torch.randint(0, P.shape[0], (n,), device="cuda", generator=g)
    cases = {
        # receiver -> random mesh vertex (deduction / first reprojection ray)
        "recv_to_mesh": (xD[ri], P[vi] - xD[ri]),
        # mesh point -> another mesh point (inner segment of a TT chain)
        "mesh_to_mesh": (P[vi], P[vj] - P[vi]),
        # random directions from receivers (mostly misses)
        "recv_random": (xD[ri], torch.randn(n, 3, device="cuda", generator=g)),
    }
    if cfg == 2:
        # walk-like rays of configs[2]: every receiver (in order: coherent) towards a point of the
        # water plane within +-0.5 of straight above it
        m = min(n, xD.shape[0])
        tgt = xD[:m].clone()
        tgt[:, 1] = 0.0
        tgt[:, 0] += torch.rand(m, device="cuda", generator=g) - 0.5
        tgt[:, 2] += torch.rand(m, device="cuda", generator=g) - 0.5
        pad = lambda a: torch.cat([a, a[: n - m]], 0) if m < n else a
        cases = {"recv_up_coherent": (pad(xD[:m]), pad(tgt - xD[:m])), **cases}
    t = torch.empty(n, device="cuda")
    prim = torch.empty(n, dtype=torch.int32, device="cuda")
    surf = torch.empty(n, dtype=torch.int32, device="cuda")
    for name, (o, d) in cases.items():
        d = d / d.norm(dim=1, keepdim=True).clamp_min(1e-20)
        O4 = torch.cat([o, torch.zeros(n, 1, device="cuda")], 1).contiguous()
        D4 = torch.cat([d, torch.zeros(n, 1, device="cuda")], 1).contiguous()
        ms = timed(lambda: mpg.mpg_trace_rays(ds.h, O4, D4, 1e-4 * ds.extent, 1, t, prim, surf))
        hit = (surf >= 0).float().mean().item()
        print(f"cfg{cfg} {name:14s} {n / ms / 1e6:8.1f} Mrays/s  ({ms:.3f} ms for {n} rays, hit {hit:.2f})")
    ds.close()


if __name__ == "__main__":
    main()
