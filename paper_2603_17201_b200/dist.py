"""Multi-GPU loop fusion: keyframe-sharded PLAN, one NCCL MIN all-reduce, replicated APPLY.

"the computations across different connected keyframes are mutually independent"
(§IV.D.3) -> the window keyframes are split into contiguous shards,
balanced by query count. Each rank runs lc_fuse(PLAN) on its shard; the winner words
(window-major) and victim words (per map point) of all ranks are merged by one
all_reduce(MIN) over a single int64 buffer -- MIN over (H << 32) | q is exactly the
lowest-(H, q) rule of the single-GPU path (readings A17, A21), so the merge is
bit-identical to FUSE_ALL on one GPU. Every rank then runs lc_fuse(APPLY) on the
whole window, so the replicated map stores stay identical without shipping them.
The map store itself is replicated (C5: ~0.6 GB of 180 GB).

Everything here is host orchestration; `fuser` is any object with Context.fuse's
signature (the CUDA Context in production, an oracle adapter in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from ._lib import LC_FUSE_APPLY, LC_FUSE_PLAN


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
                 group=None, device=None, tables=None, events=None, cur_kf=-1, forced_mp=None):
    """PLAN on this rank's shard -> all_reduce(MIN) of [winner | victim] -> APPLY.

    tables: optional preallocated int64 tensor of n_wfeat + n_mp entries on `device`
    (the NCCL buffer); events: optional (start, end) CUDA events recorded on the current
    stream around the all-reduce (the exchange's share of the step);
    returns (plan_counts, apply_counts, merged tables)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n_w = len(window)
    n_list = int(mp_list.shape[0]) if hasattr(mp_list, "shape") else len(mp_list)
    lo, hi = shard_bounds(n_w, world, win_list_begin, n_list)[rank]
    n_wfeat = fuser.n_feat_of(window)
    n_mp = fuser.n_mp
    host = device is None or torch.device(device).type == "cpu"
    if tables is None:
        tables = torch.empty(n_wfeat + n_mp, dtype=torch.int64,
                             device="cpu" if host else device)
    win, vic = tables[:n_wfeat], tables[n_wfeat:]
    w_arg = win.numpy() if host else win
    v_arg = vic.numpy() if host else vic
    extra = {} if forced_mp is None else dict(cur_kf=cur_kf, forced_mp=forced_mp)   # every rank: O9.4
    plan = fuser.fuse(window, mp_list, params, window_S=window_S, win_list_begin=win_list_begin,
                      phase=LC_FUSE_PLAN, w_lo=lo, w_hi=hi, winner=w_arg, victim=v_arg,
                      action=False, host=host, **extra)
    if events is not None:
        events[0].record()
    dist.all_reduce(tables, op=dist.ReduceOp.MIN, group=group)
    if events is not None:
        events[1].record()
    app = fuser.fuse(window, mp_list, params, window_S=window_S, win_list_begin=win_list_begin,
                     phase=LC_FUSE_APPLY, winner=w_arg, victim=v_arg, action=False, host=host)
    return plan["counts"], app["counts"], tables


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
