"""World-size-2 (and 3) gloo tests of the multi-GPU fusion protocol on CPU.

paper_2603_17201_b200.dist.fuse_sharded is run by real torch.distributed processes;
the per-rank PLAN / APPLY are served by an oracle-backed adapter with Context.fuse's
signature (the CUDA path is covered by tests/test_gpu_parity.py). The merged result
must equal the single-process oracle FUSE_ALL bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleFuser:
    """Context.fuse-compatible adapter over the CPU oracle (test infrastructure)."""

    def __init__(self, om):
        self.om = om
        self.n_mp = om.n_mp

    def n_feat_of(self, kfs):
        return self.om.window_feat_total(kfs)

    def fuse(self, window, mp_list, params, *, window_S=None, win_list_begin=None, phase=3,
             w_lo=0, w_hi=None, winner=None, victim=None, action=True, host=True, cur_kf=-1, forced_mp=None):
        return self.om.fuse(window, mp_list, params, window_S=window_S,
                            win_list_begin=win_list_begin, phase=phase, w_lo=w_lo, w_hi=w_hi,
                            winner=winner, victim=victim, cur_kf=cur_kf, forced_mp=forced_mp)

    def _gidx(self, window):
        fb = self.om.kf_feat_begin
        return np.concatenate([np.arange(fb[k], fb[k + 1]) for k in window])

    def fuse_adds_pack(self, window, w_lo, w_hi, winner, idx, word):
        """lc_fuse_adds(PACK) restated in numpy: the shard's winner words on empty slots."""
        F = np.array([self.om.n_feat_of(int(k)) for k in window])
        woff = np.r_[0, np.cumsum(F)]
        w = winner.numpy() if hasattr(winner, "numpy") else winner
        g = self._gidx(window)
        j = np.arange(woff[w_lo], woff[w_hi])
        sel = j[(w[j] != np.iinfo(np.int64).max) & (self.om.feat_mp[g[j]] == -1)]
        idx[:len(sel)] = torch.from_numpy(sel)
        word[:len(sel)] = torch.from_numpy(w[sel])
        return len(sel)

    def fuse_adds_unpack(self, window, winner, idx, word):
        winner.fill_(np.iinfo(np.int64).max)
        winner[idx] = word


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, params, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from lcsynth import make_world
    from paper_2603_17201_b200 import dist as lcdist
    w = make_world(name, 0)
    om = oracle.OracleMap(w)
    if w.win_S is None:
        om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    plan_c, app_c, info = lcdist.fuse_sharded(OracleFuser(om), w.window, w.mp_list, params,
                                              window_S=w.win_S, win_list_begin=w.win_list_begin,
                                              gather_winner=True)
    plan_sum = lcdist.sum_counts(plan_c)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), feat_mp=om.feat_mp, flags=om.mp_flags,
             rep=om.mp_replaced_by, nobs=om.mp_nobs, winner=info["winner"].numpy(),
             victim=info["victim"].numpy(), n_adds=info["n_adds"],
             cand=plan_sum["candidates"], victims=app_c["victims"])
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("T5", 2), ("C1", 2), ("T5", 3)])
def test_fuse_sharded_gloo_equals_single(tmp_path, name, world):
    import oracle
    from lcsynth import make_world
    from lcsynth.world import FUSE_PARAMS_CHECKS
    mp.spawn(_worker, args=(world, _free_port(), name, FUSE_PARAMS_CHECKS, str(tmp_path)),
             nprocs=world, join=True)
    w = make_world(name, 0)
    om = oracle.OracleMap(w)
    if w.win_S is None:
        om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    ref = om.fuse(w.window, w.mp_list, FUSE_PARAMS_CHECKS, window_S=w.win_S,
                  win_list_begin=w.win_list_begin)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["feat_mp"], om.feat_mp)
        assert np.array_equal(z["flags"], om.mp_flags)
        assert np.array_equal(z["rep"], om.mp_replaced_by)
        assert np.array_equal(z["nobs"], om.mp_nobs)
        assert np.array_equal(z["winner"], ref["winner"])
        assert np.array_equal(z["victim"], ref["victim"])
        assert int(z["n_adds"]) == ref["counts"]["add"]
        assert int(z["cand"]) == ref["counts"]["candidates"]
        assert int(z["victims"]) == ref["counts"]["victims"]


class OracleSearcher:
    def __init__(self, om):
        self.om = om

    def n_feat_of(self, kfs):
        return self.om.window_feat_total(kfs)

    def search_by_projection(self, pair_kf, pair_S, pair_param, params, pair_list_begin, mp_list,
                             pair_taken=None):
        return self.om.search_by_projection(pair_kf, pair_S, pair_param, params, pair_list_begin, mp_list,
                                            pair_taken=pair_taken)


def _search_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from lcsynth import make_world
    from lcsynth.world import SBP_PARAMS
    from paper_2603_17201_b200 import dist as lcdist
    w = make_world("C4", 0)
    fm, fd, cn = lcdist.search_sharded(OracleSearcher(oracle.OracleMap(w)), w.pair_kf, w.pair_S, w.pair_param,
                                       SBP_PARAMS, w.pair_list_begin, w.pair_mp_list, pair_taken=w.pair_taken)
    np.savez(os.path.join(out_dir, f"s{rank}.npz"), fm=fm.numpy(), fd=fd.numpy(), cn=cn.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_search_sharded_gloo_equals_single(tmp_path, world):
    """C4's 32 hypotheses x 4 pairs split across ranks (replicas of the map, pair blocks,
    all_gather of the output tables) == the single-process batched search."""
    import oracle
    from lcsynth import make_world
    from lcsynth.world import SBP_PARAMS
    mp.spawn(_search_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = make_world("C4", 0)
    ref = oracle.OracleMap(w).search_by_projection(w.pair_kf, w.pair_S, w.pair_param, SBP_PARAMS,
                                                   w.pair_list_begin, w.pair_mp_list, pair_taken=w.pair_taken)
    for r in range(world):
        z = np.load(tmp_path / f"s{r}.npz")
        assert np.array_equal(z["fm"], ref["feat_mp"]) and np.array_equal(z["fd"], ref["feat_dist"])
        assert np.array_equal(z["cn"], ref["counts"])


def test_shard_bounds_balanced_and_covering():
    from paper_2603_17201_b200.dist import shard_bounds
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        wb = np.r_[0, np.cumsum(rng.integers(0, 5000, n))]
        for W in (1, 2, 3, 4, 8):
            b = shard_bounds(n, W, wb)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(W - 1))
            loads = [wb[h] - wb[l] for l, h in b]
            assert max(loads) <= wb[-1] / W + wb[1:].__sub__(wb[:-1]).max() + 1
    assert shard_bounds(10, 4, None, 7) == [(0, 3), (3, 5), (5, 8), (8, 10)]


class OracleCorrector:
    """lc_set_point_range / lc_correct_sim3 / lc_mp_positions adapter over the CPU oracle
    (test infrastructure): a correction with a point range runs the oracle's whole
    correction and keeps the positions outside the range as they were -- the library's
    contract (poses, owners and corr_ref replicated; positions of the slice only)."""

    def __init__(self, om):
        self.om = om
        self.n_mp = om.n_mp
        self.lo, self.hi = 0, om.n_mp

    def set_point_range(self, lo=0, hi=-1):
        self.lo, self.hi = (0, self.om.n_mp) if hi < 0 else (int(lo), int(hi))

    def _slice_only(self, fn):
        before = self.om.mp_pos.copy()
        r = fn()
        keep = np.ones(self.om.n_mp, bool)
        keep[self.lo:self.hi] = False
        self.om.mp_pos[keep] = before[keep]
        return r

    def correct_window(self, cur_kf, S_cw_corr, window, host=True):
        return self._slice_only(lambda: self.om.correct_window(cur_kf, S_cw_corr, window))

    def correct_all(self, S_opt, host=True):
        return self._slice_only(lambda: self.om.correct_all(S_opt))

    def mp_positions(self, op, lo, hi, xyz, host=True):
        from paper_2603_17201_b200._lib import LC_POS_GET
        if op == LC_POS_GET:
            xyz[:] = torch.from_numpy(self.om.mp_pos[lo:hi].copy())
        else:
            self.om.mp_pos[lo:hi] = xyz.numpy()
        return xyz


def _loop_worker(rank, world, port, name, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from lcsynth import make_world
    from lcsynth.world import FUSE_PARAMS
    from paper_2603_17201_b200 import dist as lcdist
    w = make_world(name, 0)
    om = oracle.OracleMap(w)
    cor = OracleCorrector(om)
    _, nb_w = lcdist.correct_window_sharded(cor, w.cur_kf, w.S_cw_corr, w.window)
    lcdist.fuse_sharded(OracleFuser(om), w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S,
                        win_list_begin=w.win_list_begin)
    _, nb_a = lcdist.correct_all_sharded(cor, w.S_opt)
    np.savez(os.path.join(out_dir, f"l{rank}.npz"), pos=om.mp_pos, pose=om.kf_pose, feat_mp=om.feat_mp,
             nb=nb_w + nb_a)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("C1", 2), ("T5", 3)])
def test_loop_event_sharded_corrections_gloo_equal_single(tmp_path, name, world):
    """The whole loop event with the point passes of WINDOW and ALL sharded by map-point
    slice and the slices all-gathered (SURVEY.md §8(e) "Correction"), the fusion by keyframe
    shard: every rank's store == the single-process oracle's (positions, poses, associations)."""
    import oracle
    from lcsynth import make_world
    from lcsynth.world import FUSE_PARAMS
    from paper_2603_17201_b200.dist import point_bounds
    mp.spawn(_loop_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    w = make_world(name, 0)
    om = oracle.OracleMap(w)
    om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    om.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
    om.correct_all(w.S_opt)
    b = point_bounds(om.n_mp, world)
    L = max(h - l for l, h in b)
    for r in range(world):
        z = np.load(tmp_path / f"l{r}.npz")
        assert np.array_equal(z["pos"], om.mp_pos), f"rank {r}: positions"
        assert np.array_equal(z["pose"], om.kf_pose), f"rank {r}: poses"
        assert np.array_equal(z["feat_mp"], om.feat_mp), f"rank {r}: associations"
        assert int(z["nb"]) == 2 * world * L * 12


def test_point_bounds_cover():
    from paper_2603_17201_b200.dist import point_bounds
    for n in (0, 1, 7, 1000, 977802):
        for W in (1, 2, 3, 8):
            b = point_bounds(n, W)
            assert b[0][0] == 0 and b[-1][1] == n and all(b[i][1] == b[i + 1][0] for i in range(W - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
