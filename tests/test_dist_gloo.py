"""N>1 host path on CPU: world_size 2 over gloo (127.0.0.1).

Each rank walks its own partition (walk ids from dist.walk_id_base), here with
the oracle standing in for the device walk; the cross-rank operations bench.py
and a multi-GPU render use -- max-over-ranks time, summed counts, and the
walk-weighted combination of per-rank estimates (Eq. 3) -- are checked against
the same quantities computed in one process.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2311_12818_b200 import workloads as W

N_SIDE, SPP = 4, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_walks(rank):
    from oracle import oracle as O
    from paper_2311_12818_b200 import dist as D
    w = W.config0(n_side=N_SIDE, spp=SPP)
    s = O.OracleScene(w)
    base = D.walk_id_base(rank, w.n_walks)
    o = s.walks(np.arange(w.n_walks), s.opts(walk_id_base=base))
    return w, o, base


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2311_12818_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w, o, base = _rank_walks(rank)
    mean = torch.tensor(o["w"].reshape(-1, SPP).mean(1), dtype=torch.float32)
    comb = D.combine_estimates(mean, SPP)
    conv = int(np.isin(o["status"], (0, 5)).sum())
    ms, (c_sum, n_sum) = D.reduce_timing(10.0 * (rank + 1), [conv, w.n_walks])
    ids = torch.tensor([base, base + w.n_walks], dtype=torch.int64)
    gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, ids)
    if rank == 0:
        json.dump({"comb": comb.tolist(), "ms": ms, "conv": c_sum, "n": n_sum,
                   "ranges": [g.tolist() for g in gathered]}, open(out, "w"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_partition_and_reductions(tmp_path):
    out = str(tmp_path / "r.json")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = json.load(open(out))
    # partitions: disjoint, contiguous walk-id ranges
    (a0, a1), (b0, b1) = r["ranges"]
    assert a1 == b0 and a0 == 0 and b1 - b0 == a1 - a0
    # reductions against one process
    per = [_rank_walks(k)[1] for k in range(2)]
    conv = sum(int(np.isin(o["status"], (0, 5)).sum()) for o in per)
    assert r["ms"] == 20.0 and r["conv"] == conv and r["n"] == 2 * N_SIDE * N_SIDE * SPP
    ref = np.mean([o["w"].reshape(-1, SPP).mean(1) for o in per], axis=0)
    assert np.allclose(r["comb"], ref, rtol=1e-6, atol=1e-12)
    # the two partitions are different walks (independent draws), not copies
    assert not np.array_equal(per[0]["target"], per[1]["target"])


def test_single_process_is_identity():
    import torch
    from paper_2311_12818_b200 import dist as D
    m = torch.arange(5, dtype=torch.float32)
    assert torch.equal(D.combine_estimates(m, 4), m)
    assert D.reduce_timing(3.5, [1, 2]) == (3.5, [1.0, 2.0])
    assert D.walk_id_base(3, 100, base=7) == 307
