"""GPU map-point refresh (lc_refresh_mappoints) against the oracle
(O11): after a full loop event, descriptors, normals and depth bounds are compared
bit for bit (fp64 in the same order on both sides, stored fp32), with the counters."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS  # noqa: E402
from tests import tinymap as tm  # noqa: E402


@pytest.fixture(scope="module")
def Ctx():
    from paper_2603_17201_b200 import Context, build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return Context


def _compare(ctx, om):
    st = ctx.download_map()
    assert np.array_equal(st["mp_desc"], om.mp_desc), "descriptors"
    assert np.array_equal(st["mp_normal"], om.mp_normal), "normals"
    assert np.array_equal(st["mp_max_dist"], om.mp_max_dist), "depth bounds"


@pytest.mark.parametrize("name", ["T1", "T2", "C2"])
def test_refresh_after_loop_event_matches_oracle(Ctx, name):
    w = make_world(name, 0)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    for side in (ctx, om):
        side.correct_window(w.cur_kf, w.S_cw_corr, w.window)
        side.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
        side.correct_all(w.S_opt)
    # the loop's points first (the survivors of the merge), then everything
    sel = np.unique(w.mp_list).astype(np.int32)
    cg = ctx.refresh_mappoints(sel, what=3)
    co = om.refresh(sel, what=3)
    assert cg["refresh_mp"] == co["refresh_mp"] > 0 and cg["refresh_obs"] == co["refresh_obs"]
    _compare(ctx, om)
    cg = ctx.refresh_mappoints(None, what=1)
    co = om.refresh(None, what=1)
    assert cg["refresh_mp"] == co["refresh_mp"] and cg["refresh_obs"] == co["refresh_obs"]
    _compare(ctx, om)
    cg = ctx.refresh_mappoints(None, what=2)
    co = om.refresh(None, what=2)
    _compare(ctx, om)


def test_refresh_many_observations_and_skips(Ctx):
    """80 observations of one point (the global-memory path), a bad point and an
    unobserved point (both unchanged)."""
    rng = np.random.default_rng(5)
    base = rng.integers(0, 256, 32, dtype=np.uint8)
    kfs = []
    for k in range(10):
        S = tm.IDENT.copy()
        S[9:12] = -np.array([rng.uniform(-3, 3), rng.uniform(-3, 3), -5.0 - k])
        feats = [dict(u=10.0 + i, v=10.0, oct=int(rng.integers(0, 8)),
                      desc=tm.desc_with_h(base, int(rng.integers(0, 40)), offset=int(rng.integers(0, 200))),
                      mp=0 if i < 8 else (1 if i == 8 else -1)) for i in range(10)]
        kfs.append(dict(pose=S, feats=feats))
    mps = [dict(pos=(0.1, -0.2, 0.3), desc=base, ref_kf=3), dict(pos=(1.0, 1.0, 1.0), desc=base, flags=1),
           dict(pos=(2.0, 0.0, 0.0), desc=~base)]
    arrays = tm.build(kfs, mps)
    arrays["feat_mp"][arrays["feat_mp"] == 1] = 1   # point 1 is observed but bad
    ctx = Ctx(0)
    ctx.upload_map(arrays, [tm.PIN])
    om = oracle.OracleMap(arrays=arrays, cams=[tm.PIN])
    cg = ctx.refresh_mappoints(None, what=3)
    co = om.refresh(None, what=3)
    assert cg["refresh_mp"] == co["refresh_mp"] == 1 and cg["refresh_obs"] == co["refresh_obs"] == 80
    _compare(ctx, om)
    st = ctx.download_map()
    assert np.array_equal(st["mp_desc"][1], base) and np.array_equal(st["mp_desc"][2], ~base)


def _cmp_conn(g, o, max_edges):
    gn, gk, gw = g[0], g[1], g[2]
    on, ok, ow = o[0], o[1], o[2]
    assert np.array_equal(gn, on), np.nonzero(gn != on)[0][:5]
    for i in range(len(on)):
        m = min(int(on[i]), max_edges)
        assert np.array_equal(gk[i, :m], ok[i, :m]) and np.array_equal(gw[i, :m], ow[i, :m]), i


@pytest.mark.parametrize("name", ["T1", "T2", "C2"])
def test_connections_after_loop_event_match_oracle(Ctx, name):
    """Covisibility recount (lc_update_connections) after the merge:
    edge counts, keyframes and weights equal the oracle's (O12) for every keyframe."""
    w = make_world(name, 0)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    for side in (ctx, om):
        side.correct_window(w.cur_kf, w.S_cw_corr, w.window)
        side.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
    for th, me in ((15, 64), (1, 8)):
        g = ctx.update_connections(None, th=th, max_edges=me)
        o = om.update_connections(None, th=th, max_edges=me)
        _cmp_conn(g, o, me)
        assert g[3]["conn_kf"] == o[3]["conn_kf"] == w.n_kf and g[3]["conn_edges"] == o[3]["conn_edges"]
    sel = np.asarray(w.window, np.int32)
    _cmp_conn(ctx.update_connections(sel, th=15, max_edges=32), om.update_connections(sel, th=15, max_edges=32), 32)


def test_connections_spec_example_on_gpu(Ctx):
    base = tm.desc_from_bits([])
    holdings = [list(range(30)), list(range(20)) + [40, 41], list(range(25, 30)), [50]]
    kfs = [dict(feats=[dict(u=1.0 + i, v=1.0, desc=base, mp=int(q)) for i, q in enumerate(h)]) for h in holdings]
    mps = [dict(pos=(0.0, 0.0, 1.0), desc=base) for _ in range(51)]
    arrays = tm.build(kfs, mps)
    ctx = Ctx(0)
    ctx.upload_map(arrays, [tm.PIN])
    n, kf, wt, c = ctx.update_connections(None, th=5, max_edges=4)
    assert list(n) == [2, 1, 1, 0]
    assert list(kf[0, :2]) == [1, 2] and list(wt[0, :2]) == [20, 5]


def test_connections_more_edges_than_the_shared_list():
    """A keyframe covisible with 2500 others (> the 2048-edge shared list): the exact
    ranking path (weight desc, id asc) against oracle O12."""
    from paper_2603_17201_b200 import Context
    import oracle
    from tests import tinymap as tm
    n = 2500
    d = np.zeros(32, np.uint8)
    central = dict(feats=[dict(u=float(i % 400), v=float(i // 400), desc=d, mp=i) for i in range(n)])
    others = [dict(feats=[dict(u=10.0, v=10.0, desc=d, mp=i)] + ([dict(u=20.0, v=10.0, desc=d, mp=(i + 1) % n)]
                                                                  if i % 7 == 0 else [])) for i in range(n)]
    mps = [dict(pos=(0.0, 0.0, 1.0), desc=d) for _ in range(n)]
    arrays = tm.build([central] + others, mps)
    om = oracle.OracleMap(arrays=arrays, cams=[tm.PIN])
    on, okf, ow, _ = om.update_connections(None, th=1, max_edges=64)
    ctx = Context(0)
    ctx.upload_map(arrays, [tm.PIN])
    gn, gkf, gw, _ = ctx.update_connections(None, th=1, max_edges=64)
    assert on[0] == n and np.array_equal(gn, on)
    for i in range(len(on)):
        m = min(int(on[i]), 64)
        assert np.array_equal(gkf[i, :m], okf[i, :m]) and np.array_equal(gw[i, :m], ow[i, :m]), i
    ctx.close()
