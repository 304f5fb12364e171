"""GPU-vs-oracle comparison helpers for the -m gpu parity tests (tests only)."""
import numpy as np

from oracle import oracle as O


def run_gpu(w, **opt_over):
    import torch
    from paper_2311_12818_b200 import mpg
    ds = mpg.DeviceScene(w)
    b = mpg.Batch(w.xD, w.nD, w.spp, w.seed.k)
    opts = ds.opts(**opt_over)
    mpg.run_step(ds, b, opts)
    torch.cuda.synchronize()
    res = b.results()
    res["mean"] = b.mean.cpu().numpy()[:b.n_recv]
    res["var"] = b.var.cpu().numpy()[:b.n_recv]
    st = b.stats_dict()
    ext = ds.extent
    ds.close()
    return res, st, ext


def run_oracle(w, ids, **opt_over):
    s = O.OracleScene(w)
    return s.walks(np.asarray(ids, np.int64), s.opts(**opt_over)), s


def compare(g, o, ids, extent, k, w=None):
    """Walk-level parity report for walk indices `ids` (g: full GPU arrays, o: oracle on ids);
    with the workload `w`, also the triangle-id mismatches that are not shared-edge ties (R17)."""
    gs = g["status"][ids].astype(np.int64)
    os_ = o["status"].astype(np.int64)
    cg = np.isin(gs, (0, 5))
    co = np.isin(os_, (0, 5))
    both = cg & co
    rep = {"n": len(ids), "conv_gpu": int(cg.sum()), "conv_orc": int(co.sum()),
           "flag_agree": float((cg == co).mean()), "status_agree": float((gs == os_).mean()),
           "both": int(both.sum())}
    # visibility: among walks both sides converge, CONVERGED (V = 1) vs OCCLUDED (V = 0)
    rep["n_occluded_gpu"] = int((gs == 5).sum())
    rep["n_occluded_orc"] = int((os_ == 5).sum())
    rep["vis_mismatch"] = int((both & (gs != os_)).sum())
    rep["vis_agree"] = float((gs[both] == os_[both]).mean()) if both.any() else 1.0
    gp = g["pos"][ids][:, :k]
    dv = np.linalg.norm(gp - o["pos"][:, :k], axis=2)
    if "k" in o:                       # per-walk chain length (configs[4]): vertices beyond n are unused
        dv = np.where(np.arange(k)[None, :] < o["k"][:, None], dv, 0.0)
    dpos = dv.max(1)
    same = both & (dpos < 1e-4 * extent)
    rep["max_dpos_rel"] = float(dpos[same].max() / extent) if same.any() else 0.0
    rep["n_other_chain"] = int((both & ~same).sum())
    gprim = g["prim"][ids][:, :k]
    pm = gprim == o["prim"][:, :k]
    if "k" in o:
        pm |= np.arange(k)[None, :] >= o["k"][:, None]
    same_prim = pm.all(1)
    rep["prim_agree"] = float(same_prim[both].mean()) if both.any() else 1.0
    vis = (gs == 0) & (os_ == 0)
    rep["both_visible"] = int(vis.sum())
    if vis.any():
        rg = np.abs(g["G"][ids][vis] - o["G"][vis]) / np.maximum(np.abs(o["G"][vis]), 1e-30)
        rep["G_rel_med"] = float(np.median(rg))
        rep["G_rel_p99"] = float(np.quantile(rg, 0.99))
        rep["G_rel_max"] = float(rg.max())
        tr = (g["trials"][ids][vis] == o["trials"][vis])
        rep["trials_agree"] = float(tr.mean())
    if w is not None:
        rep["prim_mis"], rep["prim_bad"] = prim_mismatches(w, g, o, np.asarray(ids), extent, k)
    rep["disagree_ids"] = np.asarray(ids)[cg != co]
    rep["prim_mismatch_ids"] = np.asarray(ids)[both & ~same_prim]
    return rep


def _dist_point_segment(p, a, b):
    ab = b - a
    t = np.clip(np.dot(p - a, ab) / max(np.dot(ab, ab), 1e-300), 0.0, 1.0)
    return float(np.linalg.norm(p - (a + t * ab)))


def prim_mismatches(w, g, o, ids, extent, k, tol_rel=1e-4):
    """Reading R17: triangle ids are bit-exact on chains both sides converge to
    the same chain, except where the vertex lies on an edge (or corner) shared by the two
    triangles -- within tol_rel x extent (the position tolerance) of the shared vertices'
    segment.  Returns (mismatching vertices, list of (walk, vertex, gpu tri, oracle tri, dist)
    for mismatches that are NOT such ties)."""
    pos, _, I, _, _ = w.mesh_arrays()
    P = pos.astype(np.float64)
    gs, os_ = g["status"][ids], o["status"]
    both = np.isin(gs, (0, 5)) & np.isin(os_, (0, 5))
    n_mis, bad = 0, []
    for j in np.nonzero(both)[0]:
        kk = int(o["k"][j]) if "k" in o else k
        if np.linalg.norm(g["pos"][ids[j], :kk] - o["pos"][j, :kk], axis=1).max() > tol_rel * extent:
            continue                     # another admissible chain (counted as n_other_chain, R27)
        for v in range(kk):
            a, b = int(g["prim"][ids[j], v]), int(o["prim"][j, v])
            if a == b:
                continue
            n_mis += 1
            if a < 0 or b < 0:
                bad.append((int(ids[j]), v, a, b, np.inf))
                continue
            shared = sorted(set(I[a].tolist()) & set(I[b].tolist()))
            p = o["pos"][j, v]
            if len(shared) >= 2:
                d = _dist_point_segment(p, P[shared[0]], P[shared[1]])
            elif len(shared) == 1:
                d = float(np.linalg.norm(p - P[shared[0]]))
            else:
                d = np.inf
            if not d <= tol_rel * extent:
                bad.append((int(ids[j]), v, a, b, d / extent))
    return n_mis, bad


def tile_means(wv, spp, recv_shape, tile):
    """Per-tile (tile x tile receivers) mean and SE of w (reading R19)."""
    ny, nx = recv_shape
    a = wv.reshape(ny, nx, spp)
    ty, tx = ny // tile, nx // tile
    a = a[:ty * tile, :tx * tile].reshape(ty, tile, tx, tile, spp).transpose(0, 2, 1, 3, 4).reshape(ty * tx, -1)
    return a.mean(1), a.std(1, ddof=1), a.shape[1]


def classify_boundary(s, w, o, ids, extent, max_n=300, seed=0, offsets=None):
    """Reading R18: a flag disagreement is a basin/budget boundary case if the
    oracle's own outcome changes under one of 8 seed-target perturbations of
    1e-4 x extent, or under max_iters +- 3.  Returns (n_boundary, n_checked, non_boundary_ids).
    offsets(walk) -> [k, 2] offset uniforms of a glossy walk (R37), set for its re-runs."""
    rng = np.random.default_rng(seed)
    pos = {int(x): j for j, x in enumerate(o["walk"])}
    nb, bad = 0, []
    for i in list(ids)[:max_n]:
        j = pos[int(i)]
        if offsets is not None:
            O.set_offset_uv(offsets(int(i)))
        xD = w.xD[int(i) // w.spp].astype(np.float64)
        base = o["status"][j] in (0, 5)
        tgt = o["target"][j].astype(np.float64)
        changed = False
        for _ in range(8):
            v = rng.normal(size=3)
            v /= np.linalg.norm(v)
            r = s.walk_from_target(xD, w.nD[0], o["xL"][j], tgt + 1e-4 * extent * v)
            if (r["status"] in (0, 5)) != base:
                changed = True
                break
        if not changed:
            for mi in (w.opts.max_iters - 3, w.opts.max_iters + 3):
                r = s.walk_from_target(xD, w.nD[0], o["xL"][j], tgt, opts=s.opts(max_iters=mi))
                if (r["status"] in (0, 5)) != base:
                    changed = True
                    break
        nb += changed
        if not changed:
            bad.append(int(i))
    if offsets is not None:
        O.set_offset_uv(None)
    return nb, min(len(ids), max_n), bad
