"""Multi-GPU plumbing for the batched manifold walk (host logic only).

The walk partitions into independent walks: rank r of N walks
its own batch with walk ids [base + r*n, base + (r+1)*n) -- every random number
of a walk is drawn from its walk id (Philox counter, R13), so ranks never share
a draw and no data-path collective is needed ("scaling": "weak").  The only
cross-rank operations are measurement (max-over-ranks device time, summed
counts), for a render that spreads one receiver set over ranks, the
combination of per-rank estimates (Eq. 3 is a mean over walks, so the global
estimate is the walk-count-weighted mean of the rank means), and the one
exchange the method itself has: in the progressive loop (configs[4]) the guide
is fitted from the samples of the last iteration (P:426 footnote) --
of all ranks -- so the accumulated histograms are summed over ranks before
every rebuild; every rank then samples from the same guide.

torch.distributed carries these (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def walk_id_base(rank: int, n_per_rank: int, base: int = 0) -> int:
    """First walk id of rank `rank` (disjoint, contiguous partitions)."""
    return base + rank * n_per_rank


def reduce_timing(ms: float, counts, device=None):
    """(max over ranks of `ms`, sum over ranks of each count) -- bench's aggregation."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), [float(c) for c in counts]
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([float(x) for x in counts], dtype=torch.float64, device=device)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return float(t.item()), [float(x) for x in c.tolist()]


def combine_estimates(mean: torch.Tensor, spp: int) -> torch.Tensor:
    """Global per-receiver estimate from per-rank means over `spp` walks each:
    sum_r spp_r * mean_r / sum_r spp_r (all ranks hold the same receivers)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return mean.clone()
    num = (mean.to(torch.float64) * spp).contiguous()
    den = torch.tensor([float(spp)], dtype=torch.float64, device=mean.device)
    dist.all_reduce(num, op=dist.ReduceOp.SUM)
    dist.all_reduce(den, op=dist.ReduceOp.SUM)
    return (num / den).to(mean.dtype)


def allreduce_histogram(hist: torch.Tensor) -> torch.Tensor:
    """Sum a guide histogram over ranks in place (identity on one process)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM)
    return hist


def exchange_guide(ds, buf: torch.Tensor, stream=None):
    """Exchange step of the multi-process progressive loop (mpg.run_progressive's
    `exchange`): this rank's accumulated histogram -> buf (device, cells*types*bins
    float32) -> sum over ranks (NCCL over NVLink on the GPU box) -> back into the
    guide, before mpg_guide_rebuild."""
    from . import mpg
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return
    mpg.mpg_guide_download(ds.guide, buf, None, stream)
    allreduce_histogram(buf)
    mpg.mpg_guide_set_histogram(ds.guide, buf, stream)


def exchange_samples(ds, buf: torch.Tensor, n_local: int, stream=None):
    """Exchange step of the multi-process progressive loop with the STree + vMF guide:
    every rank's sample records of this iteration are gathered on every rank (NCCL
    all-gather; 48 B per walk), in rank order, and replace the local records before
    mpg_guide_rebuild, so every rank fits the same tree from the samples of all ranks
    (P:426 footnote).  buf: device uint8 of world * n_local * 48 bytes.

    Only the paper's default (fit from the last iteration's samples, keep_all = 0) is
    exchangeable: with keep_all the guide keeps earlier records across rebuilds, so the
    local record count is not this iteration's n_local and gathering them again would
    duplicate every earlier rank's records -- rejected up front."""
    from . import mpg
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return
    desc = getattr(ds, "stree_desc", None)
    if desc is not None and desc.keep_all:
        raise ValueError("exchange_samples: keep_all guides cannot be exchanged (records persist across rebuilds)")
    if desc is not None and desc.max_samples < dist.get_world_size() * n_local:
        raise ValueError("exchange_samples: guide capacity below world * n_local records")
    world = dist.get_world_size()
    B = mpg.GUIDE_SAMPLE_BYTES
    mine = torch.empty(n_local * B, dtype=torch.uint8, device=buf.device)
    got = mpg.mpg_guide_get_samples(ds.guide, mine, stream)
    assert got == n_local, (got, n_local)
    gather_records(mine, buf[: world * n_local * B])
    mpg.mpg_guide_set_samples(ds.guide, buf, world * n_local, stream)


def gather_records(mine: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """All-gather of equal-sized per-rank record buffers into out (rank order); NCCL or gloo."""
    world = dist.get_world_size()
    parts = list(out.view(world, -1).unbind(0))
    dist.all_gather(parts, mine)
    return out


def owner_rows(recv_z, cells_y: int, grid_origin_z: float, grid_extent_z: float, rank: int, world: int):
    """Owner-computes partition of the progressive loop: rank r owns the
    receiver rows whose guide-cell row is in [cells_y*r/world, cells_y*(r+1)/world), i.e.
    whole guide cells.  recv_z: the z coordinate of each receiver row (rows are z-major).
    A rank's walks then only ever accumulate into -- and sample from -- its own cells, so
    the histogram exchange is not needed (the tables of a rank's cells are identical with
    or without the all-reduce, tests/test_dist_gloo.py); the STree guide is fitted per rank
    from its own configurations.  Returns the owned row indices (contiguous)."""
    import numpy as np
    z = np.asarray(recv_z, np.float32)
    cz = np.floor((z - np.float32(grid_origin_z)) * np.float32(cells_y) / np.float32(grid_extent_z)).astype(np.int64)
    cz = np.clip(cz, 0, cells_y - 1)
    c0, c1 = cells_y * rank // world, cells_y * (rank + 1) // world
    return np.nonzero((cz >= c0) & (cz < c1))[0]


def owner_workload(w, rank: int, world: int):
    """This rank's share of a progressive workload under owner-computes: its receiver rows,
    spp multiplied by world (weak scaling: every rank walks as many walks per iteration as
    one GPU does on the whole receiver set)."""
    import dataclasses
    ny, nx = w.recv_shape
    zrows = w.xD.reshape(ny, nx, 3)[:, 0, 2]
    sp = w.seed
    rows = owner_rows(zrows, sp.cells_y, sp.grid_origin[1], sp.grid_extent[1], rank, world)
    sel = (rows[:, None] * nx + np.arange(nx)[None, :]).ravel() if len(rows) else np.zeros(0, np.int64)
    return dataclasses.replace(w, xD=np.ascontiguousarray(w.xD[sel]), nD=np.ascontiguousarray(w.nD[sel]),
                               spp=w.spp * world, recv_shape=(len(rows), nx)), rows
