"""A/B of the lane-per-walk kernel (MPG_POOL=0) and the warp-specialized pool kernel
(MPG_POOL=1): outputs must be bit-identical (same per-walk arithmetic, same counter-based
draws); times per walk call (CUDA events).
usage: python tools/pool_check.py [cfg ...] [--small] [--reps N]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_12818_b200 import mpg, workloads as W


def make(cfg, small):
    if cfg == 0:
        return W.config0(n_side=32 if small else 64, spp=16)
    if cfg == 1:
        return W.config1(n_side=128 if small else 1024)
    if cfg == 2:
        return W.config2(n_side=128 if small else 2048, spp=4)
    if cfg == 3:
        return W.config3(n_side=64 if small else 1024)
    raise SystemExit("cfg 0..3")


def run(ds, b, opts, pool, reps):
    os.environ["MPG_POOL"] = str(pool)
    mpg.mpg_sample_seeds(ds.h, ds.guide, ds.sampler, b.query, opts, b.seeds)
    ts = []
    for r in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mpg.mpg_manifold_walk(ds.h, ds.guide, ds.sampler, b.query, b.seeds, opts, b.out, b.stats, b.workspace)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return b.results(), b.stats_dict(), ts


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    small = "--small" in sys.argv
    reps = 3
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    only = os.environ.get("POOL_ONLY")   # "1": time the pool kernel only
    cfgs = [int(a) for a in args] or [0, 1, 2]
    bad = 0
    for cfg in cfgs:
        w = make(cfg, small)
        ds = mpg.DeviceScene(w)
        b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
        fl = w.opts.flags | 8
        if cfg >= 1:
            fl |= 4
        opts = ds.opts(flags=fl)
        t0 = time.time()
        r1, s1, t1 = run(ds, b, opts, 1, reps)
        print(f"cfg{cfg} n={b.n} pool: {['%.2f' % t for t in t1]} ms  conv={s1['converged']} newton={s1['newton_iters']} "
              f"rays={s1['rays']} trials={s1['trials']}", flush=True)
        if only:
            continue
        r0, s0, t0_ = run(ds, b, opts, 0, reps)
        print(f"cfg{cfg} n={b.n} lane: {['%.2f' % t for t in t0_]} ms  conv={s0['converged']} newton={s0['newton_iters']} "
              f"rays={s0['rays']} trials={s0['trials']}", flush=True)
        for key in ("status", "iters", "trials", "prim"):
            ne = int((r0[key] != r1[key]).sum())
            if ne:
                bad += 1
                print(f"  MISMATCH {key}: {ne}")
        conv = np.isin(r0["status"], (0, 5))
        for key in ("G", "T", "w"):
            ne = int((r0[key].view(np.uint32) != r1[key].view(np.uint32)).sum())
            if ne:
                rel = np.abs(r0[key].astype(np.float64) - r1[key]) / np.maximum(np.abs(r0[key]), 1e-30)
                print(f"  {key}: {ne} values differ in the last bits, max rel {rel.max():.2e}")
                if rel.max() > 1e-4:
                    bad += 1
        ne = int((r0["pos"][conv].view(np.uint32) != r1["pos"][conv].view(np.uint32)).sum())
        if ne:
            bad += 1
            print(f"  MISMATCH pos: {ne}")
        for f in ("walks", "converged", "newton_iters", "primary_iters", "attempts", "rays", "trials", "truncated",
                  "vertex_iters"):
            if s0[f] != s1[f]:
                print(f"  stats {f}: lane {s0[f]} pool {s1[f]}")
        print(f"cfg{cfg}: {'IDENTICAL' if not bad else 'DIFFERENT'}  speedup {min(t0_) / min(t1):.3f}x", flush=True)
        ds.close()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
