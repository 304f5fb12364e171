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


# ---- configs[4] progressive loop on 2 ranks: the guide exchange ----
def _cfg4_small():
    return W.config4(n_side=6, grid_n=32)


def _rank_hist(rank, w, s):
    """Oracle walks of this rank's partition of iteration 0 (guide reset) and
    their typed direction histogram (Eq. 9 accumulation, R22)."""
    from paper_2311_12818_b200 import dist as D
    base = D.walk_id_base(rank, w.n_walks)
    o = s.walks(np.arange(w.n_walks), s.opts(walk_id_base=base))
    return s.accumulate_dir(o["status"], o["w"], o["pos"][:, 0], o["k"], o["tau"])


def _worker_guide(rank, world, port, out):
    import hashlib
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2311_12818_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w = _cfg4_small()
    s = O.OracleScene(w)
    s.set_dir_hist(np.zeros((256, 126, 1024), np.float32))          # reset: learned branch absent
    h = torch.from_numpy(_rank_hist(rank, w, s))
    D.allreduce_histogram(h)                                          # the exchange step
    npf, tpf, dpf = O.guide_dir_tables(h.numpy())                     # every rank rebuilds from the sum
    dig = hashlib.sha256(npf.tobytes() + tpf.tobytes() + dpf.tobytes()).hexdigest()
    digs = [None] * world
    dist.all_gather_object(digs, dig)
    if rank == 0:
        np.save(out, h.numpy())
        json.dump({"digests": digs}, open(out + ".json", "w"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_progressive_guide_exchange(tmp_path):
    """Both ranks end the iteration with the same guide, fitted from the samples of
    both partitions: the summed histogram equals one process accumulating all
    walks, and the tables every rank rebuilds from it are identical."""
    from oracle import oracle as O
    out = str(tmp_path / "h.npy")
    mp.spawn(_worker_guide, args=(2, _free_port(), out), nprocs=2, join=True)
    h = np.load(out)
    digs = json.load(open(out + ".json"))["digests"]
    assert digs[0] == digs[1]
    w = _cfg4_small()
    s = O.OracleScene(w)
    s.set_dir_hist(np.zeros((256, 126, 1024), np.float32))
    ref = sum(_rank_hist(k, w, s) for k in range(2))
    assert h.sum() > 0 and np.allclose(h, ref, rtol=1e-12, atol=0)
    # each rank alone would have learned from half the samples: a different guide
    assert not np.allclose(h, _rank_hist(0, w, s))


def test_allreduce_histogram_single_process_identity():
    import torch
    from paper_2311_12818_b200 import dist as D
    h = torch.arange(6, dtype=torch.float32)
    assert torch.equal(D.allreduce_histogram(h.clone()), h)


# ---- the STree + vMF guide on 2 ranks: sample records gathered ----
def _rank_records(rank, w, s):
    """Oracle walks of this rank's partition of iteration 0 (empty tree) as sample records."""
    from oracle import oracle as O
    from paper_2311_12818_b200 import dist as D
    base = D.walk_id_base(rank, w.n_walks)
    o = s.walks(np.arange(w.n_walks), s.opts(walk_id_base=base))
    return O.record_samples(w.xD, w.spp, o["status"], o["w"].astype(np.float32), o["pos"][:, 0].astype(np.float32),
                            o["k"], o["tau"], o["xL"].astype(np.float32))


def _worker_stree(rank, world, port, out):
    import hashlib
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2311_12818_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w = W.config4(n_side=8, grid_n=32, guide="stree")
    s = O.OracleScene(w)
    mine = torch.from_numpy(np.frombuffer(_rank_records(rank, w, s).tobytes(), np.uint8).copy())
    allr = torch.empty(world * mine.numel(), dtype=torch.uint8)
    D.gather_records(mine, allr)                                       # the exchange step
    G = O.stree_build(np.frombuffer(allr.numpy().tobytes(), O.GSAMPLE))  # every rank fits from all samples
    dig = hashlib.sha256(G["nodes"].tobytes() + G["leaf_ids"].tobytes() + G["lobe_mu"].tobytes() +
                         G["lobe_prefix"].tobytes() + G["n_prefix"].tobytes()).hexdigest()
    digs = [None] * world
    dist.all_gather_object(digs, dig)
    if rank == 0:
        np.save(out, allr.numpy())
        json.dump({"digests": digs}, open(out + ".json", "w"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_stree_sample_exchange(tmp_path):
    """Both ranks fit the same STree from the records of both partitions, in rank order,
    equal to one process concatenating the two partitions' records."""
    from oracle import oracle as O
    out = str(tmp_path / "r.npy")
    mp.spawn(_worker_stree, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    digs = json.load(open(out + ".json"))["digests"]
    assert digs[0] == digs[1]
    w = W.config4(n_side=8, grid_n=32, guide="stree")
    s = O.OracleScene(w)
    ref = np.concatenate([_rank_records(k, w, s) for k in range(2)])
    assert np.array_equal(got, np.frombuffer(ref.tobytes(), np.uint8))
    assert (ref["w"] > 0).sum() > 0


def _keep_all_worker(rank, world, port, out):
    import types
    import torch
    import torch.distributed as dist
    from paper_2311_12818_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = {}
    for keep, cap in ((1, 100), (0, 10)):
        ds = types.SimpleNamespace(stree_desc=types.SimpleNamespace(keep_all=keep, max_samples=cap))
        try:
            D.exchange_samples(ds, torch.empty(0, dtype=torch.uint8), 10)
            res[f"{keep}_{cap}"] = "ok"
        except ValueError as e:
            res[f"{keep}_{cap}"] = str(e)
    if rank == 0:
        json.dump(res, open(out, "w"))
    dist.barrier()
    dist.destroy_process_group()


def test_sample_exchange_rejects_keep_all_and_small_capacity(tmp_path):
    """keep_all guides keep records across rebuilds, so gathering 'this iteration's'
    records again would duplicate them; a capacity below world * n_local would
    overflow: both are rejected before any collective."""
    out = str(tmp_path / "r.json")
    mp.spawn(_keep_all_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = json.load(open(out))
    assert "keep_all" in r["1_100"] and "capacity" in r["0_10"]


# ---- owner-computes: receiver bands aligned to guide cells, no exchange ----
def _worker_owner(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2311_12818_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w, rows = D.owner_workload(W.config4(n_side=16, grid_n=32), rank, world)
    s = O.OracleScene(w)
    s.set_dir_hist(np.zeros((256, 126, 1024), np.float32))
    base = D.walk_id_base(rank, w.n_walks)
    o = s.walks(np.arange(w.n_walks), s.opts(walk_id_base=base))
    h = s.accumulate_dir(o["status"], o["w"], o["pos"][:, 0], o["k"], o["tau"])
    summed = torch.from_numpy(h.copy())
    D.allreduce_histogram(summed)                          # what an exchange would give
    own = O.guide_dir_tables(h.astype(np.float32))
    ex = O.guide_dir_tables(summed.numpy().astype(np.float32))
    cells = sorted({int(c) for c in np.nonzero(h.reshape(256, -1).sum(1))[0]})
    np.savez(out + f".{rank}.npz", rows=rows, cells=np.array(cells), n=w.n_walks,
             own_n=own[0], own_t=own[1], own_d=own[2], ex_n=ex[0], ex_t=ex[1], ex_d=ex[2])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_owner_computes_needs_no_exchange(tmp_path):
    """Owner-computes: rank r walks the receiver rows of guide-cell rows [16r/2, 16(r+1)/2)
    with spp x 2 (weak scaling).  The bands are disjoint, cover the receivers and align to
    cell rows; each rank's histogram has mass only in its own cells, so the tables of its
    cells are bit-identical with and without the all-reduce: no data-path collective."""
    out = str(tmp_path / "o")
    mp.spawn(_worker_owner, args=(2, _free_port(), out), nprocs=2, join=True)
    r = [np.load(out + f".{k}.npz") for k in range(2)]
    rows0, rows1 = r[0]["rows"], r[1]["rows"]
    assert len(set(rows0) & set(rows1)) == 0 and sorted(np.concatenate([rows0, rows1])) == list(range(16))
    assert int(r[0]["n"]) == int(r[1]["n"]) == 8 * 16 * 2              # per-rank work = one GPU's
    for k in range(2):
        cells = r[k]["cells"]
        assert len(cells) > 0
        cy = cells // 16
        assert ((cy >= 8 * k) & (cy < 8 * (k + 1))).all()              # mass only in its own cell rows
        mine = (np.arange(256) // 16 >= 8 * k) & (np.arange(256) // 16 < 8 * (k + 1))
        for a, b in (("own_n", "ex_n"), ("own_t", "ex_t"), ("own_d", "ex_d")):
            assert np.array_equal(r[k][a][mine], r[k][b][mine])       # the exchange changes nothing it uses
