"""CUDA-graph capture (lc_graph_*, include/lc.h): a captured loop event (WINDOW
correction -> fuse -> ALL correction) replays to exactly the eager result, and the
first replay to the oracle's; every replay takes a fresh LoopSet epoch from the device
counter (two replays == two eager loop events back to back); capture misuse fails
loudly and leaves the context usable."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS, FUSE_PARAMS_CHECKS  # noqa: E402


@pytest.fixture(scope="module")
def Ctx():
    from paper_2603_17201_b200 import Context, build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return Context


def _tables(ctx, w):
    dev = torch.device("cuda:0")
    nwf = ctx.n_feat_of(w.window)
    return dict(list=torch.from_numpy(w.mp_list).to(dev), Sopt=torch.from_numpy(w.S_opt).to(dev),
                win=torch.empty(nwf, dtype=torch.int64, device=dev),
                vic=torch.empty(w.n_mp, dtype=torch.int64, device=dev))


def _loop(ctx, w, params, t):
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window, host=False)
    r = ctx.fuse(w.window, t["list"], params, window_S=w.win_S, win_list_begin=w.win_list_begin,
                 winner=t["win"], victim=t["vic"], host=False)
    ctx.correct_all(t["Sopt"], host=False)
    return r


def _snap(ctx, t, r):
    torch.cuda.synchronize()
    return (ctx.download_map(), t["win"].cpu().numpy().copy(), t["vic"].cpu().numpy().copy(),
            r["counts"].cpu().numpy().copy())


@pytest.mark.parametrize("name,params", [("T1", FUSE_PARAMS_CHECKS), ("C2", FUSE_PARAMS)])
def test_graph_replay_equals_eager_and_oracle(Ctx, name, params):
    w = make_world(name, 0)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    ctx.state_save()
    t = _tables(ctx, w)
    ref = [_snap(ctx, t, _loop(ctx, w, params, t)) for _ in range(2)]   # two eager events
    # the first event against the oracle (plain definition)
    om = oracle.OracleMap(w)
    om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    om.fuse(w.window, w.mp_list, params, window_S=w.win_S, win_list_begin=w.win_list_begin)
    om.correct_all(w.S_opt)
    assert np.array_equal(ref[0][0]["feat_mp"], om.feat_mp)
    assert np.array_equal(ref[0][0]["mp_pos"], om.mp_pos)
    assert np.array_equal(ref[0][0]["kf_pose"], om.kf_pose)

    ctx.state_restore()
    with ctx.capture() as cap:
        r = _loop(ctx, w, params, t)
    l0 = ctx.kernel_launches()
    for i in range(2):
        cap.graph.launch()
        got = _snap(ctx, t, r)
        for key in ref[i][0]:
            assert np.array_equal(got[0][key], ref[i][0][key]), (i, key)
        assert np.array_equal(got[1], ref[i][1]), (i, "winner")
        assert np.array_equal(got[2], ref[i][2]), (i, "victim")
        assert np.array_equal(got[3], ref[i][3]), (i, "counts")
    per = (ctx.kernel_launches() - l0) / 2
    assert per >= 8, per
    # replay after a restore == the first event again
    ctx.state_restore()
    cap.graph.launch()
    got = _snap(ctx, t, r)
    assert np.array_equal(got[0]["feat_mp"], ref[0][0]["feat_mp"])
    cap.graph.close()
    ctx.close()


def test_capture_misuse_fails_loudly(Ctx):
    from paper_2603_17201_b200._lib import LcError
    w = make_world("T1", 0)
    ctx = Ctx(0)
    with pytest.raises(LcError):            # no map yet
        with ctx.capture():
            pass
    ctx.upload_map(w.map_arrays(), [w.cam])
    ctx.state_save()
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)   # stored corrections (window_S may be None)
    t = _tables(ctx, w)
    with pytest.raises(LcError):            # host outputs cannot be recorded
        with ctx.capture():
            ctx.correct_all(w.S_opt)
    with pytest.raises(LcError) as e:       # pageable host data buffer: refused, capture aborted
        with ctx.capture():
            ctx.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S,
                     win_list_begin=w.win_list_begin, winner=t["win"], victim=t["vic"], host=False)
    assert e.value.status == -1
    with pytest.raises(LcError) as e:       # non-recordable call
        with ctx.capture():
            ctx.state_save()
    assert e.value.status == -2
    # the context is still usable and correct
    ctx.state_restore()
    om = oracle.OracleMap(w)
    Sg, _ = ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    So, _ = om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    assert np.array_equal(Sg, So)
    ctx.close()


def test_graph_pgo_then_all_correction(Ctx):
    """lc_pgo_sim3 inside a captured graph (its cooperative kernel and argument block are
    graph-owned), feeding lc_correct_sim3(ALL) on the device: a replay equals the eager
    calls bit for bit."""
    from lcsynth import make_pose_graph
    w = make_world("T1", 0)
    g = make_pose_graph("G0", 0)   # any graph with n_v = n_kf vertices works for the plumbing
    n = w.n_kf
    rng = np.random.default_rng(0)
    S0 = np.concatenate([g.S_init] * (n // g.n_v + 1))[:n].copy()
    E = np.stack([np.arange(n - 1), np.arange(1, n)], 1).astype(np.int32)
    M = np.stack([oracle.sim3_compose(oracle.pgo_exp(0.01 * rng.standard_normal(7)),
                                      oracle.sim3_compose(S0[j], oracle.sim3_inverse(S0[i]))) for i, j in E])
    fixed = np.zeros(n, np.uint8)
    fixed[0] = 1
    dev = torch.device("cuda:0")
    S0_d, M_d = torch.from_numpy(S0).to(dev), torch.from_numpy(M).to(dev)
    outs = []
    for mode in ("eager", "graph"):
        ctx = Ctx(0)
        ctx.upload_map(w.map_arrays(), [w.cam])
        ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
        if mode == "eager":
            S, tr, c2, cnt = ctx.pgo_sim3(S0_d, fixed, E, M_d, host=False)
            ctx.correct_all(S, host=False)
        else:
            with ctx.capture() as cap:
                S, tr, c2, cnt = ctx.pgo_sim3(S0_d, fixed, E, M_d, host=False)
                ctx.correct_all(S, host=False)
            cap.graph.launch()
        torch.cuda.synchronize()
        outs.append((S.cpu().numpy().copy(), cnt.cpu().numpy().copy(), ctx.download_map()))
        ctx.close()
    (Se, ce, me), (Sg, cg, mg) = outs
    np.testing.assert_array_equal(Se, Sg)
    np.testing.assert_array_equal(ce, cg)
    np.testing.assert_array_equal(me["kf_pose"], mg["kf_pose"])
    np.testing.assert_array_equal(me["mp_pos"], mg["mp_pos"])
