"""Multi-GPU loop fusion: keyframe-sharded PLAN, victim MIN all-reduce + sparse ADD all-gather,
replicated APPLY.

"the computations across different connected keyframes are mutually independent"
(§IV.D.3) -> the window keyframes are split into contiguous shards,
balanced by query count. Each rank runs lc_fuse(PLAN) on its shard; the victim words of
all ranks are merged by all_reduce(MIN) -- MIN over (H << 32) | q is exactly the
lowest-(H, q) rule of the single-GPU path (readings A17, A21) -- and the shards' ADDs
(winners on empty slots, the only winner words APPLY reads) travel as sparse lists, so
the merge is bit-identical to FUSE_ALL on one GPU. Every rank then runs lc_fuse(APPLY) on the
whole window, so the replicated map stores stay identical without shipping them.
The map store itself is replicated (C5: ~0.6 GB of 180 GB).

Everything here is host orchestration; `fuser` is any object with Context.fuse's
signature (the CUDA Context in production, an oracle adapter in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from ._lib import LC_FUSE_APPLY, LC_FUSE_PLAN, LC_POS_GET, LC_POS_SET


def shard_bounds(n_window: int, world: int, win_list_begin=None, n_list: int = 0):
    """Contiguous window-position shards [lo_r, hi_r) balanced by query count."""
    if win_list_begin is None:
        q = np.arange(n_window + 1, dtype=np.int64) * max(int(n_list), 1)
    else:
        q = np.asarray(win_list_begin, np.int64)
    total = q[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(q, total * r / world, side="left")))
    cuts.append(n_window)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n_window))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def fuse_sharded(fuser, window, mp_list, params, *, window_S=None, win_list_begin=None,
                 group=None, device=None, tables=None, events=None, cur_kf=-1, forced_mp=None,
                 gather_winner=False):
    """PLAN on this rank's shard -> exchange -> APPLY on every rank.

    Exchange: (1) all_reduce(MIN) of the victim words (int64 [n_mp], the cross-rank fusion
    merge: MIN of (H << 32) | q is the single-GPU rule, readings A17, A21); (2) all_gather of
    the sparse ADD lists -- (window-major feature index, winner word) of the shard's winners
    on empty slots, compacted by lc_fuse_adds(PACK) -- which APPLY needs besides the victim
    words (lc_fuse_adds(UNPACK) rebuilds the dense table it reads). APPLY is deterministic,
    so the replicated stores stay identical.

    tables: optional preallocated int64 tensor of n_wfeat + n_mp entries on `device`;
    events: optional (start, end) CUDA events recorded around the exchange;
    gather_winner: also all_gather every shard's full winner words (reporting / caller
    output; off the critical path).
    Returns (plan_counts, apply_counts, info) with info = dict(winner, victim, n_adds,
    exchange_bytes)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n_w = len(window)
    n_list = int(mp_list.shape[0]) if hasattr(mp_list, "shape") else len(mp_list)
    bounds = shard_bounds(n_w, world, win_list_begin, n_list)
    lo, hi = bounds[rank]
    n_wfeat = fuser.n_feat_of(window)
    n_mp = fuser.n_mp
    host = device is None or torch.device(device).type == "cpu"
    dev = torch.device("cpu") if host else torch.device(device)
    if tables is None:
        tables = torch.empty(n_wfeat + n_mp, dtype=torch.int64, device=dev)
    win, vic = tables[:n_wfeat], tables[n_wfeat:]
    w_arg = win.numpy() if host else win
    v_arg = vic.numpy() if host else vic
    extra = {} if forced_mp is None else dict(cur_kf=cur_kf, forced_mp=forced_mp)   # every rank: O9.4
    plan = fuser.fuse(window, mp_list, params, window_S=window_S, win_list_begin=win_list_begin,
                      phase=LC_FUSE_PLAN, w_lo=lo, w_hi=hi, winner=w_arg, victim=v_arg,
                      action=False, host=host, **extra)
    woff = np.r_[0, np.cumsum([fuser.n_feat_of([int(k)]) for k in window])]
    cap = int(max(woff[h] - woff[l] for l, h in bounds)) or 1
    shard_win = win[int(woff[lo]):int(woff[hi])].clone() if gather_winner else None
    idx = torch.empty(cap, dtype=torch.int64, device=dev)
    word = torch.empty(cap, dtype=torch.int64, device=dev)
    n = fuser.fuse_adds_pack(window, lo, hi, win, idx, word)
    if events is not None:
        events[0].record()
    dist.all_reduce(vic, op=dist.ReduceOp.MIN, group=group)
    ns = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(ns, torch.tensor([n], dtype=torch.int64, device=dev), group=group)
    ns = [int(x.item()) for x in ns]
    m = max(max(ns), 1)
    send = torch.full((2, m), -1, dtype=torch.int64, device=dev)
    send[0, :n] = idx[:n]
    send[1, :n] = word[:n]
    recv = [torch.empty((2, m), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    if events is not None:
        events[1].record()
    all_idx = torch.cat([recv[r][0, :ns[r]] for r in range(world)])
    all_word = torch.cat([recv[r][1, :ns[r]] for r in range(world)])
    fuser.fuse_adds_unpack(window, win, all_idx, all_word)
    app = fuser.fuse(window, mp_list, params, window_S=window_S, win_list_begin=win_list_begin,
                     phase=LC_FUSE_APPLY, winner=w_arg, victim=v_arg, action=False, host=host)
    full_win = None
    if gather_winner:   # the full winner table for the caller (not needed by APPLY)
        msz = cap
        pad = torch.full((msz,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
        pad[:shard_win.numel()] = shard_win
        outs = [torch.empty(msz, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        full_win = torch.cat([outs[r][:int(woff[h] - woff[l])] for r, (l, h) in enumerate(bounds)])
    info = dict(winner=full_win, victim=vic, n_adds=int(sum(ns)),
                exchange_bytes=dict(victim_allreduce=int(n_mp * 8), adds_allgather=int(world * 2 * m * 8)))
    return plan["counts"], app["counts"], info


def point_bounds(n_mp: int, world: int):
    """Contiguous map-point slices [lo_r, hi_r) of the sharded point passes (equal sizes)."""
    return [(n_mp * r // world, n_mp * (r + 1) // world) for r in range(world)]


def exchange_positions(corrector, group=None, device=None, events=None):
    """all_gather of the ranks' corrected position slices (SURVEY.md §8(e) "all_gather of
    corrected position slices"): every rank reads its slice out of its store
    (lc_mp_positions GET), the slices (padded to the largest) are all-gathered, and every
    other rank's slice is written into the local store (SET). Returns the bytes gathered."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    b = point_bounds(corrector.n_mp, world)
    L = max(max(h - l for l, h in b), 1)
    host = device is None or torch.device(device).type == "cpu"
    dev = torch.device("cpu") if host else torch.device(device)
    lo, hi = b[rank]
    send = torch.zeros((L, 3), dtype=torch.float32, device=dev)
    if hi > lo:
        corrector.mp_positions(LC_POS_GET, lo, hi, send[:hi - lo], host=host)
    recv = [torch.empty((L, 3), dtype=torch.float32, device=dev) for _ in range(world)]
    if events is not None:
        events[0].record()
    dist.all_gather(recv, send, group=group)
    if events is not None:
        events[1].record()
    for r, (l, h) in enumerate(b):
        if r != rank and h > l:
            corrector.mp_positions(LC_POS_SET, l, h, recv[r][:h - l], host=host)
    return int(world * L * 12)


def correct_window_sharded(corrector, cur_kf, S_cw_corr, window, *, group=None, device=None, events=None):
    """WINDOW correction with the point pass sharded by map-point range (SURVEY.md §8(e):
    the pose correction and owner election replicated, "point correction is sharded by MP
    index range, followed by all_gather of the slices"). Returns (counts, bytes gathered);
    the CORR_MP counter is this rank's slice."""
    rank = dist.get_rank(group)
    lo, hi = point_bounds(corrector.n_mp, dist.get_world_size(group))[rank]
    host = device is None or torch.device(device).type == "cpu"
    corrector.set_point_range(lo, hi)
    try:
        _, c = corrector.correct_window(cur_kf, S_cw_corr, window, host=host)
    finally:
        corrector.set_point_range()
    return c, exchange_positions(corrector, group=group, device=device, events=events)


def correct_all_sharded(corrector, S_opt, *, group=None, device=None, events=None):
    """ALL correction (optimised Sim3 propagation) sharded by map-point range + all_gather of
    the corrected position slices; keyframe poses replicated."""
    rank = dist.get_rank(group)
    lo, hi = point_bounds(corrector.n_mp, dist.get_world_size(group))[rank]
    host = device is None or torch.device(device).type == "cpu"
    corrector.set_point_range(lo, hi)
    try:
        c = corrector.correct_all(S_opt, host=host)
    finally:
        corrector.set_point_range()
    return c, exchange_positions(corrector, group=group, device=device, events=events)


def search_sharded(searcher, pair_kf, pair_S, pair_param, params, pair_list_begin, mp_list, *,
                   pair_taken=None, group=None, device=None):
    """Batched read-only guided search (C4: hypotheses x keyframe pairs) sharded across ranks
    (SURVEY.md §8(e) "C4: hypotheses are sharded across ranks, with all_gather of the result
    tables"): rank r searches a contiguous block of pairs balanced by query count, then the
    pair-major output tables (feat_mp, feat_dist) and per-pair counters are all_gathered, so
    every rank holds the whole batch's result. `searcher` has Context.search_by_projection's
    signature (an oracle adapter in the CPU tests). Returns (feat_mp, feat_dist, counts) as
    torch tensors on `device` (CPU when None)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    pair_kf = np.ascontiguousarray(pair_kf, np.int32)
    plb = np.ascontiguousarray(pair_list_begin, np.int64)
    n_pairs = len(pair_kf)
    bounds = shard_bounds(n_pairs, world, plb)
    lo, hi = bounds[rank]
    F = np.array([searcher.n_feat_of([int(k)]) for k in pair_kf], np.int64)
    foff = np.r_[0, np.cumsum(F)]
    sub_lb = (plb[lo:hi + 1] - plb[lo]).astype(np.int32)
    lst = mp_list[int(plb[lo]):int(plb[hi])]
    taken = None if pair_taken is None else pair_taken[int(foff[lo]):int(foff[hi])]
    dev = torch.device("cpu") if device is None else torch.device(device)
    if hi > lo:
        r = searcher.search_by_projection(pair_kf[lo:hi], np.asarray(pair_S)[lo:hi], np.asarray(pair_param)[lo:hi],
                                          params, sub_lb, lst, pair_taken=taken)
        fm, fd, cn = (torch.as_tensor(np.asarray(r[x]), device=dev) for x in ("feat_mp", "feat_dist", "counts"))
    else:
        fm = torch.zeros(0, dtype=torch.int32, device=dev)
        fd = torch.zeros(0, dtype=torch.int32, device=dev)
        cn = torch.zeros((0, 0), dtype=torch.int64, device=dev)
    mfeat = int(max(foff[h] - foff[l] for l, h in bounds)) or 1
    mpair = int(max(h - l for l, h in bounds)) or 1
    ncnt = cn.shape[1] if cn.numel() else 0
    ncnt_t = torch.tensor([ncnt], dtype=torch.int64, device=dev)
    dist.all_reduce(ncnt_t, op=dist.ReduceOp.MAX, group=group)
    ncnt = int(ncnt_t.item())
    send = torch.full((2, mfeat), -1, dtype=torch.int32, device=dev)
    send[0, :fm.numel()] = fm.to(torch.int32)
    send[1, :fd.numel()] = fd.to(torch.int32)
    sc = torch.zeros((mpair, ncnt), dtype=torch.int64, device=dev)
    if cn.numel():
        sc[:cn.shape[0]] = cn
    rf = [torch.empty_like(send) for _ in range(world)]
    rc = [torch.empty_like(sc) for _ in range(world)]
    dist.all_gather(rf, send, group=group)
    dist.all_gather(rc, sc, group=group)
    feat_mp = torch.cat([rf[r][0, :int(foff[h] - foff[l])] for r, (l, h) in enumerate(bounds)])
    feat_dist = torch.cat([rf[r][1, :int(foff[h] - foff[l])] for r, (l, h) in enumerate(bounds)])
    counts = torch.cat([rc[r][:h - l] for r, (l, h) in enumerate(bounds)])
    return feat_mp, feat_dist, counts


def sum_counts(counts, group=None, device="cpu"):
    """all_reduce(SUM) of a counts dict or tensor across ranks."""
    if isinstance(counts, dict):
        keys = list(counts)
        t = torch.tensor([counts[k] for k in keys], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return dict(zip(keys, t.tolist()))
    t = counts.clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t
