"""GPU (liblc) vs CPU oracle for the round-2 boundary additions: forced loop matches in
lc_fuse (O9.4 / A23), lc_correct_sim3(WINDOW | DRY_RUN) batches (O3', SURVEY.md §8(d)
C4), the edge-ambiguous counter (§8(c) O11) at constructed distances, and the per-keyframe
LC_UPLOAD_APPEND store against one REPLACE upload. Bars as in
test_gpu_parity.py: index tables, counters and maps bit-exact; fp64 Sim3 results and
fp32 positions bit-exact (same expression order, -fmad=false / -ffp-contract=off)."""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS, FUSE_PARAMS_CHECKS  # noqa: E402
from tests import tinymap as tm  # noqa: E402

NONE = oracle.NONE64


@functools.lru_cache(maxsize=None)
def world(name, seed=0):
    return make_world(name, seed)


@pytest.fixture(scope="module")
def Ctx():
    from paper_2603_17201_b200 import Context, build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return Context


def forced_for(w, seed=3):
    """Forced matches as detection would hand them to CorrectLoop: the loop-side twin of
    each landmark the current keyframe observes, plus 10% empty-slot ADDs."""
    c = int(w.cur_kf)
    fb = w.kf_feat_begin
    loop_mps = np.unique(np.asarray(w.mp_list, np.int64))
    lm_loop = {int(w.mp_lm[q]): int(q) for q in loop_mps}
    rng = np.random.default_rng(seed)
    forced = np.full(fb[c + 1] - fb[c], -1, np.int32)
    for f in range(len(forced)):
        m = w.feat_mp[fb[c] + f]
        if m >= 0 and int(w.mp_lm[m]) in lm_loop:
            forced[f] = lm_loop[int(w.mp_lm[m])]
        elif m < 0 and rng.random() < 0.1:
            forced[f] = int(rng.choice(loop_mps))
    return forced


@pytest.mark.parametrize("name,params", [("T1", FUSE_PARAMS), ("C1", FUSE_PARAMS_CHECKS),
                                         ("T5", FUSE_PARAMS_CHECKS), ("C2", FUSE_PARAMS)])
def test_forced_matches_parity(Ctx, name, params):
    w = world(name)
    forced = forced_for(w)
    assert (forced >= 0).sum() > 5
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    g = ctx.fuse(w.window, w.mp_list, params, window_S=w.win_S, win_list_begin=w.win_list_begin,
                 cur_kf=w.cur_kf, forced_mp=forced)
    o = om.fuse(w.window, w.mp_list, params, window_S=w.win_S, win_list_begin=w.win_list_begin,
                cur_kf=w.cur_kf, forced_mp=forced)
    assert g["counts"]["forced"] == o["counts"]["forced"] > 0
    assert np.array_equal(g["winner"], o["winner"]) and np.array_equal(g["victim"], o["victim"])
    assert np.array_equal(g["action"], o["action"])
    assert g["counts"] == o["counts"], {k: (g["counts"][k], o["counts"][k]) for k in g["counts"]
                                        if g["counts"][k] != o["counts"][k]}
    st = ctx.download_map()
    for key, ref in (("feat_mp", om.feat_mp), ("mp_flags", om.mp_flags), ("mp_replaced_by", om.mp_replaced_by),
                     ("mp_nobs", om.mp_nobs)):
        assert np.array_equal(st[key], ref), key
    ctx.close()


def _loopset_world(name="T5", n_add=6):
    """A world where reading A21 fires: victims of the base run are appended to window
    keyframe 0's loop list, so they join the LoopSet (the union of all window lists) and
    the slots they hold are never fused (loop_skip) -- the synthetic worlds alone never
    put a window slot's map point into a loop list."""
    w = world(name)
    om = oracle.OracleMap(w)
    om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    o = om.fuse(w.window, w.mp_list, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=w.win_list_begin)
    vic = np.flatnonzero(o["victim"] != NONE)[:n_add].astype(np.int32)
    assert len(vic) == n_add
    lb = np.asarray(w.win_list_begin, np.int32).copy()
    lst = np.concatenate([w.mp_list[:lb[1]], vic, w.mp_list[lb[1]:]]).astype(np.int32)
    lb[1:] += n_add
    return w, lst, lb


@pytest.mark.parametrize("mode", ["device-lists", "host-pipelined", "sole", "sharded"])
def test_loopset_skip_parity(Ctx, monkeypatch, mode):
    """Reading A21 (a slot holding a LoopSet map point is skipped, never a victim) against
    the oracle with loop_skip > 0, through the device-list, pipelined host-list (k_project
    stamps the LoopSet), sole and sharded-PLAN launches."""
    from paper_2603_17201_b200 import LC_FUSE_APPLY, LC_FUSE_PLAN
    w, lst, lb = _loopset_world()
    if mode == "host-pipelined":
        monkeypatch.setenv("LC_PIPE_MIN", "1")
    if mode == "sole":
        monkeypatch.setenv("LC_SOLE", "1")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    o = om.fuse(w.window, lst, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=lb)
    assert o["counts"]["loop_skip"] > 0
    L = lst if mode == "host-pipelined" else torch.from_numpy(lst).cuda()
    if mode == "sharded":
        cuts = np.linspace(0, len(w.window), 4).astype(int)
        tabs = [ctx.fuse(w.window, L, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=lb, phase=LC_FUSE_PLAN,
                         w_lo=cuts[r], w_hi=cuts[r + 1]) for r in range(3)]
        win = np.minimum.reduce([t["winner"] for t in tabs])
        vic = np.minimum.reduce([t["victim"] for t in tabs])
        assert sum(t["counts"]["loop_skip"] for t in tabs) == o["counts"]["loop_skip"]
        assert np.array_equal(win, o["winner"]) and np.array_equal(vic, o["victim"])
        ctx.fuse(w.window, L, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=lb, phase=LC_FUSE_APPLY,
                 winner=win, victim=vic)
    else:
        g = ctx.fuse(w.window, L, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=lb)
        assert np.array_equal(g["winner"], o["winner"]) and np.array_equal(g["victim"], o["victim"])
        assert np.array_equal(g["action"], o["action"])
        assert g["counts"] == o["counts"], {k: (g["counts"][k], o["counts"][k]) for k in g["counts"]
                                            if g["counts"][k] != o["counts"][k]}
    st = ctx.download_map()
    for key, ref in (("feat_mp", om.feat_mp), ("mp_flags", om.mp_flags), ("mp_replaced_by", om.mp_replaced_by),
                     ("mp_nobs", om.mp_nobs)):
        assert np.array_equal(st[key], ref), key
    ctx.close()


def test_forced_matches_sharded_plan_equals_fuse_all(Ctx):
    """Every shard's PLAN carries the forced matches (idempotent on an already forced map):
    PLAN per shard on one device, MIN merge, APPLY == FUSE_ALL."""
    from paper_2603_17201_b200 import LC_FUSE_APPLY, LC_FUSE_PLAN
    w = world("T5")
    forced = forced_for(w)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    ctx.state_save()
    ref = ctx.fuse(w.window, w.mp_list, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=w.win_list_begin,
                   cur_kf=w.cur_kf, forced_mp=forced)
    ref_map = ctx.download_map()
    ctx.state_restore()
    cuts = np.linspace(0, len(w.window), 4).astype(int)
    tabs = [ctx.fuse(w.window, w.mp_list, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=w.win_list_begin,
                     phase=LC_FUSE_PLAN, w_lo=cuts[r], w_hi=cuts[r + 1], cur_kf=w.cur_kf, forced_mp=forced)
            for r in range(3)]
    win = np.minimum.reduce([t["winner"] for t in tabs])
    vic = np.minimum.reduce([t["victim"] for t in tabs])
    assert np.array_equal(win, ref["winner"]) and np.array_equal(vic, ref["victim"])
    ctx.fuse(w.window, w.mp_list, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=w.win_list_begin,
             phase=LC_FUSE_APPLY, winner=win, victim=vic)
    m = ctx.download_map()
    for k in ref_map:
        assert np.array_equal(m[k], ref_map[k]), k
    ctx.close()


def test_forced_requires_window_keyframe(Ctx):
    from paper_2603_17201_b200 import _lib
    from paper_2603_17201_b200._lib import LcError
    w = world("T1")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    outside = int(np.setdiff1d(np.arange(w.n_kf), w.window)[0])
    with pytest.raises(LcError) as e:
        ctx.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=np.tile(tm.IDENT, (len(w.window), 1)),
                 cur_kf=outside, forced_mp=np.full(int(np.diff(w.kf_feat_begin)[outside]), -1, np.int32))
    assert e.value.status == _lib.LC_EINVAL
    ctx.close()


@pytest.mark.parametrize("host", [True, False], ids=["host-out", "device-out"])
def test_dry_run_batch_parity_C4(Ctx, host):
    """The 32 C4 hypotheses' window corrections as one LC_DRY_RUN batch: S_corr, the CSR of
    corrected points, their indices and fp32 positions bit-exact against oracle O3'; the
    device map is untouched (nothing written back)."""
    w = world("C4")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    before = ctx.download_map()
    om = oracle.OracleMap(w)
    oS, omb, oidx, opos, oc = om.correct_window_batch(w.hyp_cur, w.hyp_S_cw, w.hyp_win_begin, w.hyp_window)
    gS, gmb, gidx, gpos, gc = ctx.correct_window_batch(w.hyp_cur, w.hyp_S_cw, w.hyp_win_begin, w.hyp_window,
                                                       capacity=int(omb[-1]) + 7, host=host)
    if not host:
        torch.cuda.synchronize()
        n = int(gmb[-1].item())
        gS, gmb, gidx, gpos = gS.cpu().numpy(), gmb.cpu().numpy(), gidx[:n].cpu().numpy(), gpos[:n].cpu().numpy()
        gc = dict(zip(oracle.COUNTER_NAMES, gc.cpu().numpy().tolist()))
    assert np.array_equal(gS, oS)
    assert np.array_equal(gmb, omb) and np.array_equal(gidx, oidx)
    assert np.array_equal(gpos, opos)
    assert gc["corr_mp"] == oc["corr_mp"] and gc["corr_kf"] == oc["corr_kf"]
    after = ctx.download_map()
    for k in before:
        assert np.array_equal(before[k], after[k]), k
    ctx.close()


def test_dry_run_capacity_and_errors(Ctx):
    from paper_2603_17201_b200 import _lib
    from paper_2603_17201_b200._lib import LcError
    w = world("C4")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    _, omb, _, _, _ = om.correct_window_batch(w.hyp_cur[:3], w.hyp_S_cw[:3], w.hyp_win_begin[:4], w.hyp_window)
    with pytest.raises(LcError) as e:
        ctx.correct_window_batch(w.hyp_cur[:3], w.hyp_S_cw[:3], w.hyp_win_begin[:4], w.hyp_window,
                                 capacity=int(omb[-1]) - 1)
    assert e.value.status == _lib.LC_ECAPACITY
    bad = w.hyp_window.copy()
    bad[w.hyp_win_begin[1]] = bad[w.hyp_win_begin[1] + 1]      # window 1 does not start with its cur_kf
    with pytest.raises(LcError) as e:
        ctx.correct_window_batch(w.hyp_cur[:3], w.hyp_S_cw[:3], w.hyp_win_begin[:4], bad)
    assert e.value.status == _lib.LC_EINVAL
    ctx.close()


BASE = np.random.default_rng(7).integers(0, 256, 32, dtype=np.uint8)


@pytest.mark.parametrize("fu,fv,x", [
    (254.0 - 5e-5, 250.0, 0.5), (254.0 + 5e-5, 250.0, 0.5), (254.0 - 3e-4, 250.0, 0.5),
    (251.0, 246.0 + 5e-5, 0.5), (254.0 - 5e-5, 240.0, 0.5), (250.0, 250.0, 0.5),
    (1.0, 1.0, 2.0 - 4e-7), (1.0, 1.0, 2.0 - 5e-6), (1.0, 1.0, 2.0 + 4e-7), (1.0, 1.0, -2.0 + 4e-7),
])
def test_edge_counter_constructed(Ctx, fu, fv, x):
    """The library's edge-ambiguous counter equals the oracle's flag at constructed
    distances from a window edge and from the image bounds (u = 100 x + 200)."""
    p = (x, 0.5, 1.0) if x != 0.5 else (0.5, 0.5, 1.0)
    n = np.asarray(p) / np.linalg.norm(p)
    arrays = tm.build([dict(feats=[dict(u=fu, v=fv, desc=BASE)])],
                      [dict(pos=p, dmax=2.0 if x != 0.5 else 1.2, normal=tuple(n), desc=BASE)])
    om = oracle.OracleMap(arrays=arrays, cams=[tm.PIN])
    o = om.fuse([0], [0], (4, 50, 0, 0, 0), window_S=tm.IDENT[None])
    ctx = Ctx(0)
    ctx.upload_map(arrays, [tm.PIN])
    g = ctx.fuse([0], np.array([0], np.int32), (4, 50, 0, 0, 0), window_S=tm.IDENT[None])
    assert g["counts"] == o["counts"]
    ctx.close()


def _chunks(w, n_chunks):
    """Split a world's map into keyframe chunks with the map points whose reference
    keyframe falls in the chunk (map points are ordered by reference keyframe, and a point's
    observers come at or after it, so every chunk references only stored points)."""
    a = {k: np.asarray(v) for k, v in w.map_arrays().items()}
    ref = a["mp_ref_kf"]
    assert np.all(np.diff(ref) >= 0)
    fb = a["kf_feat_begin"]
    cuts = np.linspace(0, len(fb) - 1, n_chunks + 1).astype(int)
    out = []
    for k0, k1 in zip(cuts[:-1], cuts[1:]):
        m0, m1 = np.searchsorted(ref, k0), np.searchsorted(ref, k1)
        f0, f1 = fb[k0], fb[k1]
        out.append(dict(kf_pose=a["kf_pose"][k0:k1], kf_cam=a["kf_cam"][k0:k1],
                        kf_feat_begin=(fb[k0:k1 + 1] - f0).astype(np.int32),
                        feat_uv=a["feat_uv"][f0:f1], feat_octave=a["feat_octave"][f0:f1],
                        feat_angle=a["feat_angle"][f0:f1], feat_desc=a["feat_desc"][f0:f1],
                        feat_mp=a["feat_mp"][f0:f1], mp_pos=a["mp_pos"][m0:m1], mp_normal=a["mp_normal"][m0:m1],
                        mp_max_dist=a["mp_max_dist"][m0:m1], mp_desc=a["mp_desc"][m0:m1],
                        mp_angle=a["mp_angle"][m0:m1], mp_ref_kf=a["mp_ref_kf"][m0:m1],
                        mp_flags=a["mp_flags"][m0:m1]))
    return out


@pytest.mark.parametrize("name,n_chunks", [("T5", 7), ("C2", 25), ("S3", 40)])
def test_upload_append_equals_replace(Ctx, name, n_chunks):
    """PAPER.md:147-148 §IV.A ("transfer each newly created keyframe to GPU-resident
    KeyFrame Storage"): N LC_UPLOAD_APPEND calls give the store one LC_UPLOAD_REPLACE of
    the whole map gives -- downloaded state equal byte for byte, and the same loop event
    (WINDOW correction, fuse, ALL propagation) produces identical tables and maps."""
    w = world(name)
    ref = Ctx(0)
    ref.upload_map(w.map_arrays(), [w.cam])
    app = Ctx(0)
    parts = _chunks(w, n_chunks)
    app.upload_map(parts[0], [w.cam])
    for part in parts[1:]:
        app.upload_map(part, [w.cam], append=True)
    assert (app.n_kf, app.n_feat, app.n_mp) == (ref.n_kf, ref.n_feat, ref.n_mp)
    a, r = app.download_map(), ref.download_map()
    for key in r:
        assert np.array_equal(a[key], r[key]), key
    out = []
    for ctx in (app, ref):
        ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
        g = ctx.fuse(w.window, w.mp_list, FUSE_PARAMS_CHECKS, window_S=w.win_S, win_list_begin=w.win_list_begin,
                     debug=True)
        ctx.correct_all(w.S_opt)
        out.append((g, ctx.download_map()))
    (ga, ma), (gr, mr) = out
    for key in ("winner", "victim", "action", "best", "ncand"):
        assert np.array_equal(ga[key], gr[key]), key
    assert ga["counts"] == gr["counts"]
    for key in mr:
        assert np.array_equal(ma[key], mr[key]), key
    app.close()
    ref.close()


def test_upload_pinned_and_pageable_and_append_errors(Ctx):
    from paper_2603_17201_b200 import _lib
    from paper_2603_17201_b200._lib import LcError
    w = world("C2")
    arrays = w.map_arrays()
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in arrays.items()}
    c1, c2 = Ctx(0), Ctx(0)
    c1.upload_map(arrays, [w.cam])       # pageable: through the staging ring (> 1 MB arrays)
    c2.upload_map(pinned, [w.cam])       # page-locked: direct
    a, b = c1.download_map(), c2.download_map()
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    c3 = Ctx(0)
    with pytest.raises(LcError) as e:
        c3.upload_map(arrays, [w.cam], append=True)
    assert e.value.status == _lib.LC_ESTATE
    bad = _chunks(w, 2)[1]
    bad = dict(bad, feat_mp=np.full_like(bad["feat_mp"], 10 ** 7))
    c3.upload_map(_chunks(w, 2)[0], [w.cam])
    with pytest.raises(LcError) as e:
        c3.upload_map(bad, [w.cam], append=True)
    assert e.value.status == _lib.LC_ERANGE
    for c in (c1, c2, c3):
        c.close()


@pytest.mark.parametrize("name", ["C1", "T2", "C2", "C3", "S3", "C5"])
def test_loop_lists_parity(Ctx, name):
    """lc_loop_lists against oracle orc_loop_lists (ascending unique map points of each
    list's source keyframes): on the uploaded map -- where they equal the world's own lists
    -- and again after a fuse changed the associations."""
    w = world(name)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    gb, gl = ctx.loop_lists(w.list_src_begin, w.list_src_kf)
    ob, ol = om.loop_lists(w.list_src_begin, w.list_src_kf)
    assert np.array_equal(gb, ob) and np.array_equal(gl, ol)
    if w.win_list_begin is not None:
        assert np.array_equal(gb, w.win_list_begin) and np.array_equal(gl, w.mp_list)
    dev = torch.device("cuda:0")
    out = torch.empty(len(ol) + 5, dtype=torch.int32, device=dev)
    db, dl = ctx.loop_lists(w.list_src_begin, w.list_src_kf, out=out, host=False)
    torch.cuda.synchronize()
    assert np.array_equal(db, ob) and np.array_equal(dl.cpu().numpy(), ol)
    if name != "C5":
        ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
        om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
        ctx.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
        om.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
        gb, gl = ctx.loop_lists(w.list_src_begin, w.list_src_kf)
        ob, ol = om.loop_lists(w.list_src_begin, w.list_src_kf)
        assert np.array_equal(gb, ob) and np.array_equal(gl, ol)
    ctx.close()


def test_loop_lists_large_and_errors(Ctx):
    """A list over the small hash (the whole C2 map's map points: the retry with the large
    hash), empty lists, and the error paths."""
    from paper_2603_17201_b200 import _lib
    from paper_2603_17201_b200._lib import LcError
    w = world("C2")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    sb = np.array([0, 0, 150, 150, 170], np.int32)     # empty, 150 keyframes (> 6144 points), empty, 20
    sk = np.r_[np.arange(150), np.arange(200, 220)].astype(np.int32)
    gb, gl = ctx.loop_lists(sb, sk)
    ob, ol = om.loop_lists(sb, sk)
    assert gb[2] - gb[1] > 6144 and np.array_equal(gb, ob) and np.array_equal(gl, ol)
    with pytest.raises(LcError) as e:
        ctx.loop_lists([0, 1], [10 ** 6])
    assert e.value.status == _lib.LC_ERANGE
    with pytest.raises(LcError) as e:
        ctx.loop_lists(sb, sk, out=np.zeros(10, np.int32))
    assert e.value.status == _lib.LC_ECAPACITY
    ctx.close()


@pytest.mark.parametrize("name,W", [("C2", 2), ("S3", 3)])
def test_point_range_slices_equal_full_correction(Ctx, name, W):
    """lc_set_point_range + lc_mp_positions (SURVEY.md §8(e) "Correction"): W contexts, each
    correcting only its map-point slice (WINDOW, then ALL), with the slices exchanged through
    lc_mp_positions GET / SET in between and at the end, equal one context correcting every
    point -- positions, poses, and the CORR_MP counts summed over the slices. The ALL pass
    reads corr_ref, which every slice keeps for every point."""
    from paper_2603_17201_b200._lib import LC_POS_GET, LC_POS_SET
    from paper_2603_17201_b200.dist import point_bounds
    w = world(name)
    ref = Ctx(0)
    ref.upload_map(w.map_arrays(), [w.cam])
    _, c_w = ref.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    c_a = ref.correct_all(w.S_opt)
    full = ref.download_map()
    ref.close()
    b = point_bounds(w.n_mp, W)
    ctxs = []
    for r in range(W):
        c = Ctx(0)
        c.upload_map(w.map_arrays(), [w.cam])
        ctxs.append(c)

    def exchange():
        sl = [c.mp_positions(LC_POS_GET, *b[r]) for r, c in enumerate(ctxs)]
        for r, c in enumerate(ctxs):
            for r2, (l, h) in enumerate(b):
                if r2 != r:
                    c.mp_positions(LC_POS_SET, l, h, sl[r2])

    n_w = n_a = 0
    for r, c in enumerate(ctxs):
        c.set_point_range(*b[r])
        n_w += c.correct_window(w.cur_kf, w.S_cw_corr, w.window)[1]["corr_mp"]
    exchange()
    for r, c in enumerate(ctxs):
        n_a += c.correct_all(w.S_opt)["corr_mp"]
        c.set_point_range()
    exchange()
    assert n_w == c_w["corr_mp"] and n_a == c_a["corr_mp"]
    for c in ctxs:
        st = c.download_map()
        assert np.array_equal(st["mp_pos"], full["mp_pos"]) and np.array_equal(st["kf_pose"], full["kf_pose"])
        c.close()


def test_point_range_errors(Ctx):
    from paper_2603_17201_b200._lib import LC_POS_GET, LcError
    w = world("C1")
    c = Ctx(0)
    with pytest.raises(LcError):
        c.set_point_range(0, 1)   # no map
    c.upload_map(w.map_arrays(), [w.cam])
    for lo, hi in ((-1, 5), (5, 4), (0, w.n_mp + 1)):
        with pytest.raises(LcError):
            c.set_point_range(lo, hi)
        with pytest.raises(LcError):
            c.mp_positions(LC_POS_GET, lo, hi)
    with pytest.raises(LcError):
        c.mp_positions(7, 0, 1)
    assert c.mp_positions(LC_POS_GET, 3, 3).shape == (0, 3)
    c.close()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "S3", "C5"])
def test_device_offsets_lists_and_fuse(Ctx, name):
    """lc_loop_lists with a device out_begin (no host synchronisation: a scan of the counts on
    the device, the wide lists' bitmaps rebuilt at emission) == the oracle's lists; lc_fuse
    taking those device offsets (and the whole list buffer as mp_list) == lc_fuse with host
    offsets: tables, counters and the post-apply map, byte for byte."""
    w = world(name)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    ob, ol = oracle.OracleMap(w).loop_lists(w.list_src_begin, w.list_src_kf)
    db, buf = ctx.loop_lists(w.list_src_begin, w.list_src_kf, host=False, device_offsets=True)
    torch.cuda.synchronize()
    gb = db.cpu().numpy()
    assert np.array_equal(gb, ob)
    assert np.array_equal(buf[:int(gb[-1])].cpu().numpy(), ol)
    if w.window is None or len(ob) != len(w.window) + 1:   # (C1: one list shared by the window)
        ctx.close()
        return
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    ctx.state_save()
    ref = ctx.fuse(w.window, ol, FUSE_PARAMS, window_S=w.win_S, win_list_begin=ob)
    st_ref = ctx.download_map()
    ctx.state_restore()
    got = ctx.fuse(w.window, buf, FUSE_PARAMS, window_S=w.win_S, win_list_begin=db)
    st = ctx.download_map()
    assert np.array_equal(got["winner"], ref["winner"]) and np.array_equal(got["victim"], ref["victim"])
    assert got["counts"] == ref["counts"]
    for k in st:
        assert np.array_equal(st[k], st_ref[k]), k
    ctx.close()


def test_device_offsets_errors(Ctx):
    from paper_2603_17201_b200._lib import LcError
    w = world("C2")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    small = torch.empty(10, dtype=torch.int32, device="cuda:0")
    with pytest.raises(LcError):   # capacity below the lists' upper bound
        ctx.loop_lists(w.list_src_begin, w.list_src_kf, out=small, host=False, device_offsets=True)
    db, buf = ctx.loop_lists(w.list_src_begin, w.list_src_kf, host=False, device_offsets=True)
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    with pytest.raises(LcError):   # a shard's PLAN needs host offsets
        ctx.fuse(w.window, buf, FUSE_PARAMS, window_S=w.win_S, win_list_begin=db, phase=1, w_lo=0, w_hi=3)
    with pytest.raises(LcError):   # so do the per-query debug outputs
        ctx.fuse(w.window, buf, FUSE_PARAMS, window_S=w.win_S, win_list_begin=db, debug=True)
    ctx.close()


def test_point_range_does_not_touch_dry_runs_and_forced_needs_host_offsets(Ctx):
    """A point range set for a sharded correction does not restrict LC_DRY_RUN batches (they
    write no positions: the whole batch is returned); a fuse with device list offsets
    refuses forced matches (their LoopSet must be stamped before the search)."""
    from paper_2603_17201_b200._lib import LcError
    w = world("C4")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    ref = ctx.correct_window_batch(w.hyp_cur, w.hyp_S_cw, w.hyp_win_begin, w.hyp_window)
    ctx.set_point_range(0, w.n_mp // 3)
    got = ctx.correct_window_batch(w.hyp_cur, w.hyp_S_cw, w.hyp_win_begin, w.hyp_window)
    ctx.set_point_range()
    for a_, b_ in zip(ref[:4], got[:4]):
        assert np.array_equal(a_, b_)
    ctx.close()
    w = world("C2")
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    db, buf = ctx.loop_lists(w.list_src_begin, w.list_src_kf, host=False, device_offsets=True)
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    forced = np.full(int(w.kf_feat_begin[w.cur_kf + 1] - w.kf_feat_begin[w.cur_kf]), -1, np.int32)
    with pytest.raises(LcError):
        ctx.fuse(w.window, buf, FUSE_PARAMS, window_S=w.win_S, win_list_begin=db, cur_kf=int(w.cur_kf),
                 forced_mp=forced)
    ctx.close()
