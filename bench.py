#!/usr/bin/env python3
"""bench.py -- batched manifold walk throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1]

A step is one pass of the whole hot path over one batch of synthetic input
(SURVEY §8(a)): light samples + guided/initial seeds (mpg_sample_seeds) ->
deduction, Newton with ray-traced reprojection, validation, kappa/G/T and
reciprocal-probability trials (mpg_manifold_walk) -> per-pixel estimator
(mpg_estimate) [-> guide accumulation for guided configs].  The workload is
BASELINE.json configs[2] (16,777,216 k=1 walks through the water heightfield, the
largest configuration that fits one GPU; BASELINE.json's metric names none) unless
--config says otherwise.  N>1: one process per GPU (torchrun), each rank walks
its own independent partition (walk_id_base = rank*n); no data-path collective.

Prints ONE JSON line (rank 0).  --impl reference times the oracle (the plain
CPU implementation in oracle/, single-threaded) on a bounded sample.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "converged manifold walks/s"
CONFIG_NAMES = {0: "configs[0]: k=1 mirror sphere, 64x64 receivers x 16 cap seeds (65,536 walks)",
                1: "configs[1]: k=2 TT glass icosphere (5,120 tris), 1024x1024 receivers x 1 seed (1,048,576 walks)",
                2: "configs[2]: k=1 T water heightfield (522,242 tris), 2048x2048 receivers x 4 guided seeds (16,777,216 walks)",
                3: "configs[3]: k=6 TTTTTT three bumpy glass slabs (780,300 tris), 1024x1024 receivers, guided seeds (1,048,576 walks)",
                4: "configs[4]: mixed scene (mirror sphere + glass icosphere + water), n in 1..6 and type per sample, "
                   "typed 16x16x126x32x32 direction guide, 8 progressive iterations x 1,048,576 walks"}

# algorithmic FP32 work per unit: a Newton vertex evaluation
# (constraint + 3 Jacobian blocks + block-Thomas step) and the ray-casting units
FLOP_PER_VERTEX_SWEEP = 540.0
FLOP_PER_NODE = 40.0
FLOP_PER_TRI = 40.0
# FP32 peak from unit counts and the max SM clock (B200_PROFILING.md: 148 SMs,
# 128 FP32 lanes/SM, FMA = 2 flops, clocks.max.sm 1965 MHz)
def fp32_peak_tflops(sm_mhz=1965.0, sms=148):
    return sms * 128 * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, idx=0):
        self.idx = idx
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[3 + j].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_workload(cfg, guide="hist"):
    from paper_2311_12818_b200 import workloads as W
    if cfg == 4:
        return W.config4(guide=guide)
    return W.CONFIGS[cfg]()


def oracle_rate(w, n_walks, seed_base=0):
    """Time the oracle (oracle/, plain single-threaded C) on the first n_walks."""
    from oracle import oracle as O
    s = O.OracleScene(w)
    ids = np.arange(n_walks, dtype=np.int64)
    t0 = time.perf_counter()
    r = s.walks(ids, s.opts(walk_id_base=seed_base))
    dt = time.perf_counter() - t0
    conv = int(np.isin(r["status"], (0, 5)).sum())
    return conv / dt, dt, conv, int(r["total_iters"].sum())


def _oracle_shard(args):
    cfg, lo, hi, seed_base, barrier, trials = args
    from oracle import oracle as O
    w = make_workload(cfg)
    s = O.OracleScene(w)
    ids = np.arange(lo, hi, dtype=np.int64)
    if barrier is not None:
        barrier.wait()
    t0 = time.perf_counter()
    r = s.walks(ids, s.opts(walk_id_base=seed_base, trials=int(trials)))
    t1 = time.perf_counter()
    return int(np.isin(r["status"], (0, 5)).sum()), int(r["total_iters"].sum()), t0, t1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate_parallel(cfg, n_walks, procs, seed_base=0, trials=True):
    """The oracle (single-threaded C) on the first n_walks, split into `procs`
    contiguous shards run by that many worker processes on the host cores.
    Scene/BVH builds are excluded (workers start timing together after a barrier).
    Returns (converged/s, wall s, converged, Newton iterations)."""
    import multiprocessing as mpr
    procs = max(1, min(procs, n_walks))
    if procs == 1:
        c, it, t0, t1 = _oracle_shard((cfg, 0, n_walks, seed_base, None, trials))
        return c / (t1 - t0), t1 - t0, c, it
    ctx = mpr.get_context("spawn")   # the ours-arm parent holds a CUDA context: never fork it
    bar = ctx.Manager().Barrier(procs)
    cuts = np.linspace(0, n_walks, procs + 1).astype(np.int64)
    with ctx.Pool(procs) as pool:
        res = pool.map(_oracle_shard, [(cfg, int(cuts[i]), int(cuts[i + 1]), seed_base, bar, trials)
                                       for i in range(procs)])
    c = sum(r[0] for r in res)
    it = sum(r[1] for r in res)
    dt = max(r[3] for r in res) - min(r[2] for r in res)
    return c / dt, dt, c, it


def host_procs():
    return max(1, min(os.cpu_count() or 1, 64))


def cpu_baseline(args, w):
    """The oracle as it stands on the host cores (SURVEY 8(d) Timing): (ii) all cores
    (one single-threaded process per core on contiguous shards), trials on = the
    reported value, and trials off; (i) one core on the first walks, trials on / off."""
    P = host_procs()
    n = min(w.n_walks, args.ref_walks * P)
    v, dt, conv, it = oracle_rate_parallel(args.config, n, P)
    v0, dt0, conv0, it0 = oracle_rate_parallel(args.config, n, P, trials=False)
    n1 = min(w.n_walks, args.ref_walks_single)
    v1, dt1, conv1, it1 = oracle_rate_parallel(args.config, n1, 1)
    v10, dt10, _, it10 = oracle_rate_parallel(args.config, n1, 1, trials=False)
    return {"value": v, "unit": "walks/s", "cores": P, "kind": "oracle", "cpu_model": cpu_model(),
            "newton_iters_per_s": it / dt,
            "sample": f"first {n} walks of the workload, {P} single-threaded oracle processes on "
                      f"contiguous shards ({dt:.1f} s wall, {conv} converged), trials on",
            "all_cores_trials_off": {"value": v0, "newton_iters_per_s": it0 / dt0, "walks": n, "wall_s": dt0},
            "single_core_trials_on": {"value": v1, "newton_iters_per_s": it1 / dt1, "walks": n1, "wall_s": dt1},
            "single_core_trials_off": {"value": v10, "newton_iters_per_s": it10 / dt10, "walks": n1,
                                       "wall_s": dt10}}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    w = make_workload(args.config)
    P = host_procs()
    n = min(w.n_walks, args.ref_walks * P)
    for _ in range(args.warmup):
        oracle_rate(w, 64)
    vals, dts, its = [], [], []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        v, dt, conv, iters = oracle_rate_parallel(args.config, n, P)
        vals.append(v)
        dts.append(dt)
        its.append(iters / dt)
    wall = time.perf_counter() - t_all
    value = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "walks/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[args.config], "sample_walks_per_step": n},
            "newton_iters_per_s": float(np.mean(its)),
            "cpu_baseline": {"value": value, "unit": "walks/s", "cores": P, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"first {n} walks of the workload per step (of {w.n_walks}), "
                                       f"{P} single-threaded oracle processes on contiguous shards"},
            "e2e": {"value": value, "unit": "walks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2311_12818_b200 import mpg
    from paper_2311_12818_b200 import dist as D
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = make_workload(args.config, args.guide)
    progressive = w.seed.mode in (3, 4)  # configs[4]: one step = the whole 8-iteration loop (R22)
    stree = w.seed.mode == 4             # --guide stree: the paper's STree + vMF guide
    iters = 8 if progressive else 1
    # N > 1 progressive loop: owner-computes by default -- each rank walks the
    # receiver rows of its guide-cell rows with spp x N, fits its guide from its own samples
    # and exchanges nothing; --exchange keeps every rank on all receivers with the guide
    # exchange (histogram all-reduce / STree record all-gather)
    owner = progressive and world > 1 and not args.exchange
    if owner:
        w, _ = D.owner_workload(w, rank, world)
    # independent partitions (weak scaling): rank r owns walk ids [r*n*iters, (r+1)*n*iters)
    w.opts.walk_id_base = D.walk_id_base(rank, w.n_walks * iters)
    ds = mpg.DeviceScene(w, stree_capacity=max(w.n_walks, args.photons) * world)
    b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
    fl = (w.opts.flags | (4 if args.f64 else 0) | (0 if args.no_sort else 8)) & ~(4 if args.f32 else 0)
    opts = ds.opts(flags=fl)
    stream = torch.cuda.current_stream()
    guided = ds.guide is not None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2


    # configs[4] on N ranks: the guide histogram is summed over ranks before every
    # rebuild (the method's one exchange step); no-op on one rank
    gsz = ds.info_guide_size() if (progressive and not stree) else 0
    hbuf = torch.empty(max(gsz, 1), dtype=torch.float32, device=dev)
    exchange = None
    if progressive and world > 1 and not owner:
        if stree:   # STree: the sample records of all ranks are gathered (the tree is fitted from all of them)
            sbuf = torch.empty(b.n * world * mpg.GUIDE_SAMPLE_BYTES, dtype=torch.uint8, device=dev)
            exchange = lambda d: D.exchange_samples(d, sbuf, b.n)
        else:
            exchange = lambda d: D.exchange_guide(d, hbuf)

    plane = (w.xD[0].tolist(), w.nD[0].tolist())   # receiver plane (photon landing, R33)

    pbuf = None
    if stree and args.photons and world > 1 and not owner:
        pbuf = torch.empty(args.photons * world * mpg.GUIDE_SAMPLE_BYTES, dtype=torch.uint8, device=dev)

    def photon_init():
        if stree and args.photons:      # photon-based p_0: iteration 0 from photons
            ex = (lambda d: D.exchange_samples(d, pbuf, args.photons)) if pbuf is not None else None
            mpg.photon_init(ds, args.photons, plane[0], plane[1], seed=1, base=rank * args.photons, exchange=ex)

    def step():
        if progressive:
            mpg.mpg_guide_reset(ds.guide)
            photon_init()
            mpg.run_progressive(ds, b, opts, iterations=iters, exchange=exchange, reset=False)
        else:
            mpg.run_step(ds, b, opts, accumulate=guided)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # the FP32 roof of this GPU, measured here (FFMA microbenchmark), before the timed region
    measured_peak = mpg.mpg_measure_fp32_peak() if not args.nominal_peak else None

    # ---- device-timed region: K steps, L2 flushed before each (outside the events) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    stats = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    wall0 = time.perf_counter()
    launches0 = mpg.mpg_kernel_launches()
    walk_ev = []
    part_ev = []
    for i in range(args.steps):
        flush.fill_(float(i))
        e0, e1, e2, e3 = ev[i]
        e0.record(stream)
        if progressive:
            mpg.mpg_guide_reset(ds.guide)
            photon_init()
        base = opts.walk_id_base
        for it in range(iters):
            opts.walk_id_base = base + it * b.n
            ev5 = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            ev5[0].record(stream)
            mpg.mpg_sample_seeds(ds.h, ds.guide, ds.sampler, b.query, opts, b.seeds)
            ev5[1].record(stream)
            mpg.mpg_manifold_walk(ds.h, ds.guide, ds.sampler, b.query, b.seeds, opts, b.out, b.stats, b.workspace)
            ev5[2].record(stream)
            walk_ev.append((ev5[1], ev5[2]))
            mpg.mpg_estimate(b.w, b.n_recv, b.spp, b.mean, b.var)
            ev5[3].record(stream)
            if stree:
                mpg.mpg_guide_record_samples(ds.guide, b.query, b.seeds, b.out, b.n)
            elif guided:
                mpg.mpg_guide_accumulate(ds.guide, b.query, b.out, b.n)
            if progressive:
                if exchange is not None:
                    exchange(ds)
                mpg.mpg_guide_rebuild(ds.guide)
            ev5[4].record(stream)
            part_ev.append(ev5)
            stats.append(b.stats.clone())
        opts.walk_id_base = base
        e1.record(stream)
        e2.record(stream)
        e3.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = mpg.mpg_kernel_launches() - launches0     # libmpg kernels enqueued in the timed region
    clk = clocks.stop()
    step_ms = [ev[i][0].elapsed_time(ev[i][3]) for i in range(args.steps)]
    walk_ms_all = [a.elapsed_time(z) for a, z in walk_ev]
    parts = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(4)] for e in part_ev]).sum(0) / args.steps
    walk_ms = [sum(walk_ms_all[i * iters:(i + 1) * iters]) for i in range(args.steps)]
    seed_ms = [0.0] * args.steps
    tot_ms = sum(step_ms)
    st = torch.stack(stats).cpu().numpy().astype(np.int64)
    fields = mpg.STATS_FIELDS
    S = {f: int(st[:, j].sum()) for j, f in enumerate(fields)}
    conv_total = S["converged"]
    tot_ms, (conv_all, newton_all) = D.reduce_timing(tot_ms, [conv_total, S["newton_iters"]], device=dev)
    value = conv_all / (tot_ms / 1e3)

    # ---- roofline of the dominant kernel (k_walk): ALU bound ----
    walk_s = sum(walk_ms) / 1e3
    flops = (FLOP_PER_VERTEX_SWEEP * S["vertex_iters"] + FLOP_PER_NODE * S["node_visits"] +
             FLOP_PER_TRI * S["tri_tests"])
    achieved = flops / walk_s / 1e12
    peak = measured_peak if measured_peak else fp32_peak_tflops()
    traffic = None
    ncu_units = None     # what the committed ncu capture of this config's k_walk says limits it
    prof = os.path.join(ROOT, "profiles", f"ncu_walk_cfg{args.config}.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic = pj.get("dram_bytes_per_launch")
            ncu_units = {"source": f"profiles/ncu_walk_cfg{args.config}.json (ncu --set full, one k_walk launch)",
                         "l1_data_pipe_lsu_wavefronts_pct_of_peak": pj.get("l1_data_pipe_lsu_wavefronts_pct_of_peak"),
                         "issue_active_pct": pj.get("issue_active_pct"),
                         "active_threads_per_warp_instruction": pj.get("simt_threads_per_inst"),
                         "dram_throughput_pct": pj.get("dram_throughput_pct"),
                         "top_stalls_pct": pj.get("top_stalls_pct")}
        except Exception:
            traffic = None

    # ---- compulsory HBM traffic of a step: seeds, walk I/O, estimator ----
    per_walk = ((16 + 16) / w.spp          # x_D, n_D read by the walk (per receiver)
                + 16 / w.spp               # x_D read by the seed kernel
                + 2 * (16 + 16 + 4 + (8 if progressive else 0))   # seeds written, then read (x_L, target, bin[, ctype, P(n)])
                + 16 * w.seed.k + 1 + 2 + 12 + 4 + (2 if progressive else 0)   # chain, status, iters, G/T/w, trials[, ctype]
                + 4 + 8 / w.spp)           # estimator: w in, mean/var out
    hbm_bytes = per_walk * b.n * iters
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm_peak = 6533.8          # MEASURED_PEAKS.json figure for this pool (copy-bandwidth, GB/s)
    hbm_gbs = hbm_bytes / (tot_ms / args.steps / 1e3) / 1e9
    hbm = {"bytes_per_step": int(hbm_bytes), "achieved_gbs": hbm_gbs, "peak_gbs": hbm_peak,
           "frac": hbm_gbs / hbm_peak, "what": "compulsory I/O per step (inputs, seeds, outputs, estimate)"}

    # ---- end to end through the public API: pinned host in -> device -> host result ----
    e2e = None
    if not args.no_e2e:
        xh, nh = b.xD_host, b.nD_host
        out_h = torch.empty(b.n_recv, dtype=torch.float32, pin_memory=True)
        for _ in range(2):
            b.xD.copy_(xh, non_blocking=True); b.nD.copy_(nh, non_blocking=True)
            step(); out_h.copy_(b.mean[:b.n_recv], non_blocking=True)
        torch.cuda.synchronize()
        e_ms = []
        conv_e = 0
        for i in range(args.steps):
            flush.fill_(float(i))
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            b.xD.copy_(xh, non_blocking=True)
            b.nD.copy_(nh, non_blocking=True)
            step()
            out_h.copy_(b.mean[:b.n_recv], non_blocking=True)
            s1.record(stream)
            s1.synchronize()
            e_ms.append(s0.elapsed_time(s1))
            conv_e += conv_total // args.steps      # the walks are deterministic: same count every step
        te = sum(e_ms)
        te, (conv_e,) = D.reduce_timing(te, [conv_e], device=dev)
        e2e = {"value": conv_e / (te / 1e3), "unit": "walks/s",
               "h2d_bytes_per_step": int(xh.numel() * 4 + nh.numel() * 4),
               "d2h_bytes_per_step": int(out_h.numel() * 4), "ms_per_step": te / args.steps}

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, w)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "walks/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64" if opts.flags & 4 else "f32", "data": "synthetic",
                "config": {"workload": CONFIG_NAMES[args.config] + (
                               " -- guide: STree over (x_D, x_L) + per-type vMF mixtures (SURVEY 8(f)1) in place of "
                               "the histogram" if stree else "") + (
                               f"; iteration 0 from {args.photons} photons (SURVEY 8(f)4)" if stree and args.photons
                               else ""), "n_walks_per_gpu": b.n, "k": w.seed.k,
                           "max_iters": w.opts.max_iters, "trials": "on (k_max 1024)",
                           "l2": "256 MB buffer written before every timed step (inputs < 126 MB L2)",
                           "order": ("primaries in walk order" if not opts.flags & 8 else
                                     "primaries in (receiver cell, seed direction) order, MPG_FLAG_SORT"),
                           "path": "persistent kernel",
                           "parallelism": (f"{world} ranks, owner-computes receiver bands aligned to guide-cell rows, "
                                           "spp x N, no data-path collective" if owner else
                                           f"{world} ranks, disjoint walk-id partitions" +
                                           (", guide exchange per iteration" if progressive and world > 1 else "")),
                           "bvh": (f"{ds.info.bvh_width}-wide SAH, {ds.info.n_nodes} nodes, {ds.info.n_tri} triangles"
                                   if ds.info.n_tri else "analytic surfaces only"),
                           "precision": ("fp32 scene/traversal; fp64 positions, residual, hit refinement" +
                                         ("; fp64 Jacobian/step (MPG_FLAG_NEWTON_F64)" if opts.flags & 4
                                          else "; fp32 Jacobian/step"))},
                "newton_iters_per_s": newton_all / (tot_ms / 1e3),
                "walks_incl_trials_per_s": S["attempts"] * world / (tot_ms / 1e3),
                "rays_per_s": S["rays"] * world / (tot_ms / 1e3),
                "breakdown_ms": {"seeds": float(parts[0]), "walk": float(parts[1]), "estimate": float(parts[2]),
                                 "accumulate+tables": float(parts[3])},
                "per_walk_time": {   # rates per second of mpg_manifold_walk time
                    "primary_converged_walks_per_s": conv_all / (sum(walk_ms) / 1e3),
                    "walks_incl_trials_per_s": S["attempts"] * world / (sum(walk_ms) / 1e3),
                    "newton_iters_per_s": newton_all / (sum(walk_ms) / 1e3)},
                "roofline": {"bound": "alu", "kernel": "k_walk", "achieved": achieved, "peak": peak,
                             "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                             "peak_source": ("measured in this run: FFMA microbenchmark (mpg_measure_fp32_peak, "
                                             "8 independent chains per thread, SMs x 4 x 256 threads, best of 5)"
                                             if measured_peak else
                                             "148 SM x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md unit counts)"),
                             "nominal_peak": fp32_peak_tflops(),
                             "algorithmic_flops_per_launch": flops / args.steps,
                             "ncu_units": ncu_units},
                "hbm": hbm,
                "stats_per_step": {k: v / args.steps for k, v in S.items()},
                "gpu_launches": launches,
                "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "wall_s_timed_region": wall}
        print(json.dumps(line), flush=True)
    ds.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--ref-walks", type=int, default=200000, help="oracle walks per host process (cpu_baseline)")
    ap.add_argument("--ref-walks-single", type=int, default=65536, help="oracle walks of the single-core timing")
    ap.add_argument("--nominal-peak", action="store_true", help="roofline against the unit-count FP32 peak")
    ap.add_argument("--guide", default="hist", choices=["hist", "stree"],
                    help="configs[4] guide: BASELINE's histogram (default) or the paper's STree + vMF (SURVEY 8(f)1)")
    ap.add_argument("--photons", type=int, default=0,
                    help="with --guide stree: photon-based initial guide from this many photons (SURVEY 8(f)4)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sort", action="store_true",
                    help="walk-order primaries (default: coherence-sorted order, MPG_FLAG_SORT; same results)")
    ap.add_argument("--exchange", action="store_true",
                    help="N>1 progressive loop: all receivers on every rank + guide exchange (default: owner-computes)")
    ap.add_argument("--f64", action="store_true", help="MPG_FLAG_NEWTON_F64")
    ap.add_argument("--f32", action="store_true", help="clear MPG_FLAG_NEWTON_F64 (fp32 Jacobian/step)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
