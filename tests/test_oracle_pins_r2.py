"""Pins of the oracle parts added in round 2 (SURVEY.md §8(c) Table B style): the forced
loop matches of the current keyframe (O9.4, reading A23), the batched dry-run window
correction (O3'), the orientation bin mapping (A15), the
edge-ambiguity flag (§8(c) "Edge-ambiguous") and the timing-only grid PLAN. Each pin is
an independent restatement (hand-built expected maps, closed forms, invariants) rather
than a re-call of the oracle's own routine. No GPU needed.
"""
import numpy as np
import pytest

import oracle
from tests import tinymap as tm

BASE = np.random.default_rng(7).integers(0, 256, 32, dtype=np.uint8)
P0 = (0.5, 0.5, 1.0)     # projects exactly to (250, 250) under tm.PIN
NONE = oracle.NONE64


def _unit(p):
    p = np.asarray(p, np.float64)
    return tuple(p / np.linalg.norm(p))


def _mp(pos=P0, dmax=1.2, normal=None, desc=BASE, flags=0, angle=0.0):
    return dict(pos=pos, dmax=dmax, normal=normal if normal is not None else _unit(pos),
                desc=desc, flags=flags, angle=angle)


FAR = (0.5, 0.5, -1.0)   # behind every camera: never matched by the search


# ----------------------------------------------------------- O9.4 forced loop matches
def test_forced_matches_constructed_cases():
    """EXT CorrectLoop: for each current-keyframe feature with a loop-matched map point q,
    the slot's occupant is replaced by q (Replace: all its observations move to q) or q is
    added to an empty slot -- before the search, which then sees q as already found."""
    # MPs: 0 A (non-loop, also seen by KF1), 1 L0 (loop), 2 L1 (loop), 3 L2 (loop, already
    # in cur f2), 4 B (in the loop list -> never a victim), 5 bad, 6 L3 (loop, bad)
    mps = [_mp(pos=FAR), _mp(pos=FAR), _mp(pos=FAR), _mp(pos=FAR), _mp(pos=FAR),
           _mp(pos=FAR, flags=1), _mp(pos=FAR, flags=1)]
    cur = dict(feats=[dict(u=10.0, v=10.0, desc=BASE, mp=0),      # f0: A   <- forced L0: A victim
                      dict(u=20.0, v=10.0, desc=BASE),            # f1: empty <- forced L1: ADD
                      dict(u=30.0, v=10.0, desc=BASE, mp=3),      # f2: L2  <- forced L2: nothing
                      dict(u=40.0, v=10.0, desc=BASE, mp=4),      # f3: B   <- forced L0: B in LoopSet
                      dict(u=50.0, v=10.0, desc=BASE, mp=5),      # f4: bad <- forced L1: nothing
                      dict(u=60.0, v=10.0, desc=BASE)])           # f5: empty <- forced L3 (bad): nothing
    kf1 = dict(feats=[dict(u=10.0, v=10.0, desc=BASE, mp=0),      # A -> rewired to L0
                      dict(u=20.0, v=10.0, desc=BASE, mp=2)])     # L1
    om = oracle.OracleMap(arrays=tm.build([cur, kf1], mps), cams=[tm.PIN])
    forced = np.array([1, 2, 3, 1, 2, 6], np.int32)
    loop_list = [1, 2, 3, 4, 6]
    out = om.fuse([0, 1], loop_list, (4, 50, 0, 0, 0), window_S=np.stack([tm.IDENT, tm.IDENT]),
                  cur_kf=0, forced_mp=forced)
    c = out["counts"]
    assert c["forced"] == 2                       # one victim (A), one ADD (L1 on f1)
    assert om.feat_mp.tolist() == [1, 2, 3, 4, 5, -1, 1, 2]
    assert om.mp_flags[0] & 1 and om.mp_replaced_by[0] == 1
    assert om.mp_nobs.tolist() == [0, 2, 2, 1, 1, 1, 0]
    assert c["victims"] == 1 and c["rewired"] == 2 and c["added"] == 1 and c["dup_cleared"] == 0
    # the search sees the updated map: every loop point held by its keyframe is "found"
    # (KF0 holds L0, L1, L2, B; KF1 holds L0, L1; the bad L3 is skipped in both)
    assert c["skip_found"] == 4 + 2 and c["skip_bad"] == 2 and c["proposals"] == 0


def test_forced_duplicate_slot_kept_by_priority():
    """A forced ADD of q on f1 while q already sits in f3 of the same keyframe: the
    pre-existing slot (priority 0) keeps q, the ADD (priority 1) is cleared (A22)."""
    mps = [_mp(pos=FAR), _mp(pos=FAR)]
    cur = dict(feats=[dict(u=10.0, v=10.0, desc=BASE), dict(u=20.0, v=10.0, desc=BASE),
                      dict(u=30.0, v=10.0, desc=BASE), dict(u=40.0, v=10.0, desc=BASE, mp=1)])
    om = oracle.OracleMap(arrays=tm.build([cur], mps), cams=[tm.PIN])
    out = om.fuse([0], [1], (4, 50, 0, 0, 0), window_S=tm.IDENT[None], cur_kf=0,
                  forced_mp=np.array([-1, 1, -1, -1], np.int32))
    assert om.feat_mp.tolist() == [-1, -1, -1, 1] and out["counts"]["dup_cleared"] == 1


def _ext_replace(arr, cur_kf, forced, loopset):
    """Independent restatement of EXT CorrectLoop's forced fusion on a host copy of the
    map arrays (MapPoint::Replace semantics adapted by readings A20-A22): returns the
    expected (feat_mp, flags, replaced_by)."""
    fb = arr["kf_feat_begin"]
    fm = arr["feat_mp"].copy()
    flags = arr["mp_flags"].copy()
    rep = np.full(len(flags), -1, np.int32)
    f0 = fb[cur_kf]
    victims, adds = {}, {}
    for f, q in enumerate(forced):
        if q < 0 or flags[q] & 1:
            continue
        m = fm[f0 + f]
        if m == q:
            continue
        if m < 0:
            adds[f0 + f] = q
        elif flags[m] & 1 or loopset[m]:
            continue
        else:
            victims[m] = q
    # new value + priority per slot, then per keyframe the least (priority, slot) keeps a point
    new = fm.copy()
    pri = np.zeros(len(fm), np.int32)
    for s in range(len(fm)):
        if fm[s] >= 0 and fm[s] in victims:
            new[s], pri[s] = victims[fm[s]], 2
        elif s in adds:
            new[s], pri[s] = adds[s], 1
    for k in range(len(fb) - 1):
        seen = {}
        for s in sorted(range(fb[k], fb[k + 1]), key=lambda s: (pri[s], s)):
            if new[s] < 0:
                continue
            if new[s] in seen:
                new[s] = -1
            else:
                seen[new[s]] = s
    for m, q in victims.items():
        flags[m] |= 1
        rep[m] = q
    return new, flags, rep


def test_forced_matches_equal_ext_replace_on_synthetic_world():
    """On T1: forced matches = the loop-side twin of every landmark the current keyframe
    observes (what detection's SearchByProjection hands CorrectLoop), plus 10% empty-slot
    ADDs. Running the forced step with an empty loop search must equal the independent
    EXT-Replace restatement, and fuse(forced) must equal fuse() on that pre-fused map."""
    from lcsynth import make_world
    w = make_world("T1", 0)
    arr = {k: np.array(v) for k, v in w.map_arrays().items()}
    c = int(w.cur_kf)
    fb = arr["kf_feat_begin"]
    loop_mps = np.asarray(w.mp_list, np.int64)
    lm_loop = {int(w.mp_lm[q]): int(q) for q in loop_mps}
    rng = np.random.default_rng(3)
    forced = np.full(fb[c + 1] - fb[c], -1, np.int32)
    for f in range(len(forced)):
        m = arr["feat_mp"][fb[c] + f]
        if m >= 0 and int(w.mp_lm[m]) in lm_loop:
            forced[f] = lm_loop[int(w.mp_lm[m])]
        elif m < 0 and rng.random() < 0.1:
            forced[f] = int(rng.choice(loop_mps))
    assert (forced >= 0).sum() > 20
    loopset = np.zeros(w.n_mp, bool)
    loopset[loop_mps] = True
    exp_fm, exp_flags, exp_rep = _ext_replace(arr, c, forced, loopset)
    # (a) forced step alone: the search list is the loop list but no window keyframe can
    # match (window_S flips every point behind the camera)
    om = oracle.OracleMap(w)
    S = np.tile(tm.IDENT, (len(w.window), 1))
    S[:, 8] = -1.0
    S[:, 4] = -1.0
    out = om.fuse(w.window, w.mp_list, (4, 50, 0, 0, 0), window_S=S, cur_kf=c, forced_mp=forced)
    assert out["counts"]["proposals"] == 0 and out["counts"]["forced"] > 20
    assert np.array_equal(om.feat_mp, exp_fm)
    assert np.array_equal(om.mp_flags, exp_flags)
    assert np.array_equal(om.mp_replaced_by, exp_rep)
    assert np.array_equal(om.mp_nobs, np.bincount(exp_fm[exp_fm >= 0], minlength=w.n_mp))
    # (b) with the real search: fuse(forced) == fuse() on the pre-fused map
    om1 = oracle.OracleMap(w)
    om1.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    o1 = om1.fuse(w.window, w.mp_list, (4, 50, 0, 0, 0), window_S=w.win_S,
                  win_list_begin=w.win_list_begin, cur_kf=c, forced_mp=forced)
    # (EXT order: CorrectLoop corrects the window first, then fuses the forced matches,
    # then runs SearchAndFuse -- so the restated map is edited after the correction)
    om2 = oracle.OracleMap(w)
    om2.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    om2.feat_mp[:] = exp_fm
    om2.mp_flags[:] = exp_flags
    om2.mp_replaced_by[:] = exp_rep
    om2.mp_nobs[:] = np.bincount(exp_fm[exp_fm >= 0], minlength=w.n_mp)
    o2 = om2.fuse(w.window, w.mp_list, (4, 50, 0, 0, 0), window_S=w.win_S, win_list_begin=w.win_list_begin)
    assert np.array_equal(o1["winner"], o2["winner"]) and np.array_equal(o1["victim"], o2["victim"])
    assert np.array_equal(om1.feat_mp, om2.feat_mp)
    assert np.array_equal(om1.mp_flags, om2.mp_flags)
    assert np.array_equal(om1.mp_replaced_by, om2.mp_replaced_by)
    assert np.array_equal(om1.mp_nobs, om2.mp_nobs)
    # (c) idempotent (a second PLAN on the same map -- a sharded one-device run -- changes
    # nothing more) and forced = all -1 is the plain fuse
    before = om.feat_mp.copy()
    out = om.fuse(w.window, w.mp_list, (4, 50, 0, 0, 0), window_S=S, cur_kf=c, forced_mp=forced, phase=1)
    # (the only re-proposals are ADDs of a point the keyframe already holds elsewhere,
    # cleared again by the priority rule)
    assert out["counts"]["forced"] == out["counts"]["dup_cleared"] and np.array_equal(om.feat_mp, before)
    assert out["counts"]["victims"] == 0
    om3, om4 = oracle.OracleMap(w), oracle.OracleMap(w)
    for o in (om3, om4):
        o.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    a = om3.fuse(w.window, w.mp_list, (4, 50, 0, 0, 0), win_list_begin=w.win_list_begin, window_S=w.win_S,
                 cur_kf=c, forced_mp=np.full_like(forced, -1))
    b = om4.fuse(w.window, w.mp_list, (4, 50, 0, 0, 0), win_list_begin=w.win_list_begin, window_S=w.win_S)
    assert np.array_equal(a["winner"], b["winner"]) and np.array_equal(om3.feat_mp, om4.feat_mp)


def test_forced_requires_cur_kf_in_window():
    from lcsynth import make_world
    w = make_world("T1", 0)
    om = oracle.OracleMap(w)
    outside = int(np.setdiff1d(np.arange(w.n_kf), w.window)[0])
    with pytest.raises(ValueError):
        om.fuse(w.window, w.mp_list, (4, 50, 0, 0, 0), window_S=np.tile(tm.IDENT, (len(w.window), 1)),
                cur_kf=outside, forced_mp=np.full(om.n_feat_of(outside), -1, np.int32))


# ------------------------------------------------------------ O3' batched dry runs
def _batches(w, n):
    rng = np.random.default_rng(5)
    cur, S, wb, win = [], [], [0], []
    for b in range(n):
        c = int(rng.choice(w.window))
        others = [int(k) for k in rng.choice(np.setdiff1d(np.arange(w.n_kf), [c]), 3, replace=False)]
        cur.append(c)
        D = tm.random_sim3(rng)
        D[9:12] *= 0.05
        D[12] = 1.0 + 0.02 * rng.standard_normal()
        S.append(oracle.sim3_compose(w.kf_pose[c], D))
        win += [c] + others
        wb.append(len(win))
    return np.array(cur, np.int32), np.stack(S), np.array(wb, np.int32), np.array(win, np.int32)


def test_dry_run_batch_invariants():
    """Every output point equals inverse(S_cw^corr) o T_cw^old (p) -- the O3 invariant makes
    the corrected position independent of the owner (1e-6 relative, fp32 storage); the
    point set is the non-bad points the batch's window observes (numpy set algebra);
    S_corr = T_iw T_wc S_cw^corr by 4x4 products; nothing is written back."""
    from lcsynth import make_world
    w = make_world("T1", 0)
    om = oracle.OracleMap(w)
    before = {k: getattr(om, k).copy() for k in ("kf_pose", "mp_pos", "mp_corr_ref", "kf_in_window")}
    cur, S, wb, win = _batches(w, 6)
    Sc, mb, idx, pos, cnt = om.correct_window_batch(cur, S, wb, win)
    for k, v in before.items():
        assert np.array_equal(getattr(om, k), v), k
    fb = w.kf_feat_begin
    assert cnt["corr_kf"] == len(win) and cnt["corr_mp"] == mb[-1]
    for b in range(len(cur)):
        ks = win[wb[b]:wb[b + 1]]
        obs = np.concatenate([w.feat_mp[fb[k]:fb[k + 1]] for k in ks])
        obs = np.unique(obs[obs >= 0])
        obs = obs[(w.mp_flags[obs] & 1) == 0]
        assert np.array_equal(idx[mb[b]:mb[b + 1]], obs), b
        c = cur[b]
        Mc = np.linalg.inv(tm.to_mat4(S[b])) @ tm.to_mat4(w.kf_pose[c])
        for j in range(mb[b], mb[b + 1]):
            p = np.r_[w.mp_pos[idx[j]].astype(np.float64), 1.0]
            exp = (Mc @ p)[:3]
            np.testing.assert_allclose(pos[j], exp, rtol=1e-6, atol=1e-6)
        for i, k in enumerate(ks):
            np.testing.assert_allclose(tm.to_mat4(Sc[wb[b] + i]),
                                       tm.to_mat4(w.kf_pose[k]) @ np.linalg.inv(tm.to_mat4(w.kf_pose[c]))
                                       @ tm.to_mat4(S[b]), atol=1e-9)


def test_dry_run_identity_and_capacity():
    from lcsynth import make_world
    w = make_world("T1", 0)
    om = oracle.OracleMap(w)
    cur, S, wb, win = _batches(w, 3)
    S_id = np.stack([w.kf_pose[c] for c in cur])          # S_cw^corr = T_cw: no correction
    Sc, mb, idx, pos, _ = om.correct_window_batch(cur, S_id, wb, win)
    np.testing.assert_allclose(pos, w.mp_pos[idx], rtol=2e-7, atol=1e-6)
    np.testing.assert_allclose(Sc, w.kf_pose[win], atol=1e-12)
    with pytest.raises(OverflowError):
        om.correct_window_batch(cur, S, wb, win, capacity=int(mb[-1]) - 1)
    bad = win.copy()
    bad[wb[1]] = (cur[1] + 1) % w.n_kf                    # window must start with cur_kf
    with pytest.raises(ValueError):
        om.correct_window_batch(cur, S, wb, bad)


# ------------------------------------------------------------ A15 bin mapping
def test_orientation_bins_round_wrap_and_12_degree_width():
    """Reading A15: bin = lround(rot * 30/360) with 30 -> 0 (12-degree bins), rot = angle_f -
    angle_q (+360 if negative). Constructed so that floor() instead of lround, 30-degree
    bins (the EXT factor quirk) or a missing wrap all change which winner is rejected:
      A 10 x rot 0          -> bin 0 (every rule)
      E 1 x rot -6 -> 354   -> 29.5 -> 30 -> wrap -> bin 0   (floor: 29, 30-deg: 12)
      B 2 x rot 90          -> 7.5 -> 8                      (floor: 7,  30-deg: 3)
      F 1 x rot 270         -> 22.5 -> 23                    (floor: 22, 30-deg: 9)
    Ours: bins {0: 11, 8: 2, 23: 1} -> max3 = 1 < 0.1 * 11 -> F rejected, E kept.
    floor or 30-degree bins: {0: 10, x: 2, y: 1, z: 1} -> max3 = 1 >= 1.0 -> F kept, E dropped."""
    rots = [(0.0, 0.0)] * 10 + [(10.0, 16.0)] + [(90.0, 0.0)] * 2 + [(270.0, 0.0)]
    feats, mps = [], []
    rng = np.random.default_rng(11)
    for j, (fa, qa) in enumerate(rots):
        u = 60.0 + 20.0 * j
        d = rng.integers(0, 256, 32, dtype=np.uint8)
        feats.append(dict(u=u, v=250.0, desc=d, angle=fa))
        p = ((u - 200.0) / 100.0, 0.5, 1.0)
        mps.append(_mp(pos=p, desc=d, dmax=float(np.linalg.norm(p)), angle=qa))
    om = oracle.OracleMap(arrays=tm.build([dict(feats=feats)], mps), cams=[tm.PIN])
    out = om.fuse([0], list(range(len(rots))), (4, 50, 0, 0, 1), window_S=tm.IDENT[None])
    assert out["counts"]["winners"] == 14 and out["counts"]["orient_rej"] == 1
    assert out["action"][13] == 4 and out["action"][10] == 1      # F rejected, E (wrapped) kept
    assert om.feat_mp[10] == 10 and om.feat_mp[13] == -1


# ------------------------------------------------------------ edge-ambiguity flag
@pytest.mark.parametrize("fu,fv,edge", [
    (254.0 - 5e-5, 250.0, 1),      # |du| = r - 5e-5: inside, within 1e-4 of the edge
    (254.0 + 5e-5, 250.0, 1),      # outside, within 1e-4
    (254.0 - 3e-4, 250.0, 0),      # inside, 3e-4 from the edge
    (254.0 + 3e-4, 250.0, 0),      # outside, 3e-4 from the edge
    (251.0, 246.0 + 5e-5, 1),      # |dv| = r - 5e-5
    (254.0 - 5e-5, 240.0, 0),      # du near the edge but |dv| far outside: not a window decision
    (250.0, 250.0, 0),
])
def test_edge_flag_window(fu, fv, edge):
    om = oracle.OracleMap(arrays=tm.build([dict(feats=[dict(u=fu, v=fv, desc=BASE)])], [_mp()]), cams=[tm.PIN])
    r = om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))
    assert r["status"] == 0 and r["edge"] == edge
    out = om.fuse([0], [0], (4, 50, 0, 0, 0), window_S=tm.IDENT[None])
    assert out["counts"]["edge_amb"] == edge


@pytest.mark.parametrize("x,edge", [(2.0 - 4e-7, 1), (2.0 - 5e-6, 0), (2.0 + 4e-7, 1), (-2.0 + 4e-7, 1)])
def test_edge_flag_bounds(x, edge):
    """u = 100 x + 200 against [0, 400): within 1e-4 px of a bound -> edge (4e-7 m = 4e-5 px)."""
    om = oracle.OracleMap(arrays=tm.build([dict(feats=[dict(u=1.0, v=1.0, desc=BASE)])],
                                          [_mp(pos=(x, 0.0, 1.0), dmax=2.0)]), cams=[tm.PIN])
    assert om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))["edge"] == edge


# ------------------------------------------------------------ grid PLAN (timing only)
@pytest.mark.parametrize("name", ["C1", "T2", "T5"])
@pytest.mark.parametrize("checks", [False, True])
def test_grid_plan_equals_brute_force(name, checks):
    """bench.py's CPU baseline (cell grid, threads) computes the same tables and counters
    as the brute-force definition (edge_amb is not evaluated in grid mode)."""
    from lcsynth import make_world
    from lcsynth.world import FUSE_PARAMS, FUSE_PARAMS_CHECKS
    w = make_world(name, 0)
    prm = FUSE_PARAMS_CHECKS if checks else FUSE_PARAMS
    om = oracle.OracleMap(w)
    om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    o = om.fuse(w.window, w.mp_list, prm, window_S=w.win_S, win_list_begin=w.win_list_begin, phase=1)
    g = om.grid()
    for t in (1, 3):
        r = om.fuse_plan_grid(g, t, w.window, w.mp_list, prm, window_S=w.win_S, win_list_begin=w.win_list_begin)
        assert np.array_equal(o["winner"], r["winner"]) and np.array_equal(o["victim"], r["victim"])
        co, cg = dict(o["counts"]), dict(r["counts"])
        co.pop("edge_amb"), cg.pop("edge_amb")
        assert co == cg


# ------------------------------------------------------------ loop map-point lists
@pytest.mark.parametrize("name", ["C1", "T5", "C2"])
def test_loop_lists_equal_set_union(name):
    """The loop list of a window keyframe is the ascending unique union of its source
    keyframes' map points; restated with numpy set algebra."""
    from lcsynth import make_world
    w = make_world(name, 0)
    om = oracle.OracleMap(w)
    ob, ol = om.loop_lists(w.list_src_begin, w.list_src_kf)
    fb = w.kf_feat_begin
    for l in range(len(ob) - 1):
        ks = w.list_src_kf[w.list_src_begin[l]:w.list_src_begin[l + 1]]
        s = np.concatenate([w.feat_mp[fb[k]:fb[k + 1]] for k in ks])
        assert np.array_equal(ol[ob[l]:ob[l + 1]], np.unique(s[s >= 0])), l
    if w.win_list_begin is not None:   # the world's own lists
        assert np.array_equal(ob, w.win_list_begin) and np.array_equal(ol, w.mp_list)
    else:
        assert np.array_equal(ol, w.mp_list)


def test_loop_lists_duplicates_bad_and_empty():
    d = np.zeros(32, np.uint8)
    kfs = [dict(feats=[dict(u=1.0, v=1.0, desc=d, mp=m) for m in ms]) for ms in ([3, 1, -1], [1, 2], [], [4])]
    mps = [dict(pos=(0.0, 0.0, 1.0), desc=d, flags=(1 if i == 2 else 0)) for i in range(5)]
    om = oracle.OracleMap(arrays=tm.build(kfs, mps), cams=[tm.PIN])
    ob, ol = om.loop_lists([0, 2, 3, 3, 5], [0, 1, 2, 2, 3])
    assert ob.tolist() == [0, 3, 3, 3, 4]
    assert ol.tolist() == [1, 2, 3, 4]      # bad point 2 included (the queries skip it, O4)
