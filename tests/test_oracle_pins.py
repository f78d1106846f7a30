"""Pins of the CPU oracle against things fixed outside of it (SURVEY.md §8(c) Table B):
values printed in the spec examples, closed forms, invariants, brute force on tiny
inputs, hand-built boundary cases, and synthetic ground truth. No GPU needed.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests import tinymap as tm

GOLD = os.path.join(os.path.dirname(__file__), "golden")
rng0 = np.random.default_rng(12345)


def _popcount_bytes(a, b):
    # independent: big-integer popcount of the XOR
    return bin(int.from_bytes(bytes(np.bitwise_xor(a, b)), "little")).count("1")


# --------------------------------------------------------------------------- O1
def test_hamming_invariants():
    rng = np.random.default_rng(1)
    for _ in range(300):
        a, b, c = (rng.integers(0, 256, 32, dtype=np.uint8) for _ in range(3))
        assert oracle.hamming(a, a) == 0
        assert oracle.hamming(a, ~a) == 256
        assert oracle.hamming(a, b) == oracle.hamming(b, a)
        assert oracle.hamming(a, b) == _popcount_bytes(a, b)
        assert oracle.hamming(a, c) <= oracle.hamming(a, b) + oracle.hamming(b, c)
    z = np.zeros(32, np.uint8)
    for bit in range(256):
        assert oracle.hamming(z, tm.desc_from_bits([bit])) == 1


# --------------------------------------------------------------------------- O2
def test_sim3_algebra_against_homogeneous_matrices():
    rng = np.random.default_rng(2)
    for _ in range(1000):
        A, B = tm.random_sim3(rng), tm.random_sim3(rng)
        AB = oracle.sim3_compose(A, B)
        np.testing.assert_allclose(tm.to_mat4(AB), tm.to_mat4(A) @ tm.to_mat4(B), rtol=0, atol=1e-12)
        Ai = oracle.sim3_inverse(A)
        np.testing.assert_allclose(tm.to_mat4(oracle.sim3_compose(A, Ai)), np.eye(4), atol=1e-12)
        np.testing.assert_allclose(tm.to_mat4(oracle.sim3_compose(Ai, A)), np.eye(4), atol=1e-12)
    for _ in range(20):
        A, B = tm.random_sim3(rng), tm.random_sim3(rng)
        p = rng.standard_normal(3)
        np.testing.assert_allclose(oracle.sim3_apply(oracle.sim3_compose(A, B), p),
                                   oracle.sim3_apply(A, oracle.sim3_apply(B, p)), atol=1e-12)
        np.testing.assert_allclose(oracle.sim3_apply(A, p), (tm.to_mat4(A) @ np.r_[p, 1])[:3],
                                   atol=1e-12)


def test_sim3_inverse_of_pure_scale_and_se3():
    S = tm.IDENT.copy()
    S[12] = 2.0
    Si = oracle.sim3_inverse(S)
    assert Si[12] == 0.5 and np.all(Si[:9] == tm.IDENT[:9]) and np.all(Si[9:12] == 0)
    rng = np.random.default_rng(3)
    for _ in range(50):
        A = tm.random_sim3(rng)
        p = rng.standard_normal(3)
        # SE3 part (R, t/s) acts as S/s: pixels are invariant to s (reading A2)
        np.testing.assert_allclose(oracle.sim3_apply(oracle.sim3_se3(A), p),
                                   oracle.sim3_apply(A, p) / A[12], atol=1e-12)


def test_scale_table():
    st = oracle.scale_table(8, 1.2)
    assert st[0] == 1.0
    np.testing.assert_allclose(st, 1.2 ** np.arange(8), rtol=1e-15)


# ------------------------------------------------------------------ projection
def test_pinhole_golden_known_pixels():
    g = json.load(open(os.path.join(GOLD, "pinhole_known_pixels.json")))
    cam = dict(model=0, k=(0, 0, 0, 0), min_x=0, max_x=640, min_y=0, max_y=480, **g["camera"])
    for c in g["cases"]:
        np.testing.assert_allclose(oracle.project(cam, c["p"]), c["uv"], atol=1e-12)


def test_pinhole_unproject_roundtrip():
    from lcsynth import CAMERAS
    cam = CAMERAS["euroc"]
    rng = np.random.default_rng(4)
    for _ in range(200):
        u, v = rng.uniform(0, cam.width), rng.uniform(0, cam.height)
        z = rng.uniform(0.5, 20)
        p = [(u - cam.cx) * z / cam.fx, (v - cam.cy) * z / cam.fy, z]
        np.testing.assert_allclose(oracle.project(cam, p), [u, v], atol=1e-9)


def test_kb8_axis_equidistant_and_roundtrip():
    from lcsynth import CAMERAS
    kb = CAMERAS["tumvi"]
    np.testing.assert_allclose(oracle.project(kb, [0, 0, 3.0]), [kb.cx, kb.cy], atol=0)
    # k = 0: equidistant model r = f * theta (textbook closed form)
    eq = dict(model=1, fx=200.0, fy=200.0, cx=256.0, cy=256.0, k=(0, 0, 0, 0),
              min_x=0, max_x=512, min_y=0, max_y=512)
    for th_deg, phi_deg in [(30, 0), (45, 90), (60, 200), (80, 315)]:
        th, phi = math.radians(th_deg), math.radians(phi_deg)
        p = [math.sin(th) * math.cos(phi), math.sin(th) * math.sin(phi), math.cos(th)]
        uv = oracle.project(eq, p)
        np.testing.assert_allclose(uv, [256 + 200 * th * math.cos(phi), 256 + 200 * th * math.sin(phi)],
                                   atol=1e-9)
    # general k: Newton unprojection of a pixel, then projection returns it
    rng = np.random.default_rng(5)
    k1, k2, k3, k4 = kb.k
    for _ in range(100):
        rad, ang = rng.uniform(1, 230), rng.uniform(0, 2 * math.pi)   # theta < 90 deg
        u, v = kb.cx + rad * math.cos(ang), kb.cy + rad * math.sin(ang)
        mx, my = (u - kb.cx) / kb.fx, (v - kb.cy) / kb.fy
        rr = math.hypot(mx, my)
        th = rr
        for _ in range(50):
            f = th * (1 + k1 * th**2 + k2 * th**4 + k3 * th**6 + k4 * th**8) - rr
            df = 1 + 3 * k1 * th**2 + 5 * k2 * th**4 + 7 * k3 * th**6 + 9 * k4 * th**8
            th -= f / df
        z = rng.uniform(0.5, 5)
        p = [math.sin(th) * mx / rr * z / math.cos(th), math.sin(th) * my / rr * z / math.cos(th), z]
        np.testing.assert_allclose(oracle.project(kb, p), [u, v], atol=1e-9)


def test_predict_level_matches_log_form():
    rng = np.random.default_rng(6)
    n = 0
    while n < 2000:
        d = rng.uniform(0.3, 20)
        dmax = d * math.exp(rng.uniform(-1, 2.5))
        x = math.log(dmax / d) / math.log(1.2)
        if abs(x - round(x)) < 1e-9:
            continue
        expect = min(max(math.ceil(x), 0), 7)
        assert oracle.predict_level(d, dmax) == expect, (d, dmax)
        n += 1


# --------------------------------------------------------------- query culls
def _one_kf_map(feats, mps):
    return oracle.OracleMap(arrays=tm.build([dict(feats=feats)], mps), cams=[tm.PIN])


def _unit(p):
    p = np.asarray(p, np.float64)
    return tuple(p / np.linalg.norm(p))


BASE = np.random.default_rng(7).integers(0, 256, 32, dtype=np.uint8)
P0 = (0.5, 0.5, 1.0)     # projects exactly to (250, 250) under tm.PIN
D0 = math.sqrt(1.5)


def _mp(pos=P0, dmax=1.2, normal=None, desc=BASE, flags=0, angle=0.0):
    return dict(pos=pos, dmax=dmax, normal=normal if normal is not None else _unit(pos),
                desc=desc, flags=flags, angle=angle)


def test_query_exact_projection_identical_descriptor():
    om = _one_kf_map([dict(u=250.0, v=250.0, desc=BASE)], [_mp()])
    r = om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))
    assert r["status"] == 0 and r["u"] == 250.0 and r["v"] == 250.0
    assert r["level"] == 0 and r["radius"] == 4.0
    assert (r["ncand"], r["best_f"], r["best_h"], r["second_h"]) == (1, 0, 0, 256)


@pytest.mark.parametrize("pos,status", [
    ((0.5, 0.5, -1.0), oracle.Q_DEPTH), ((0.5, 0.5, 0.0), oracle.Q_DEPTH),
    ((3.0, 0.0, 1.0), oracle.Q_BOUNDS), ((2.0, 0.0, 1.0), oracle.Q_BOUNDS),   # u = 400 (half-open)
    ((-2.0, 0.0, 1.0), 0), ((0.0, -2.0, 1.0), 0),                             # u or v = 0 kept
])
def test_query_depth_and_bounds(pos, status):
    om = _one_kf_map([dict(u=1.0, v=1.0, desc=BASE)], [_mp(pos=pos, dmax=2.0)])
    assert om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))["status"] == status


def test_query_distance_range_and_view_angle():
    prm = (4, 50, 0, 0, 0)
    z = 2.0
    for dmax, st in [(z / 1.2 * 1.01, 0), (z / 1.2 * 0.99, oracle.Q_DIST),
                     (z * 1.2 ** 7 / 0.8 * 0.99, 0), (z * 1.2 ** 7 / 0.8 * 1.01, oracle.Q_DIST)]:
        om = _one_kf_map([dict(u=200.0, v=200.0, desc=BASE)], [_mp(pos=(0, 0, z), dmax=dmax)])
        assert om.query(0, tm.IDENT, 0, prm)["status"] == st, dmax
    for ang, st in [(59.0, 0), (61.0, oracle.Q_ANGLE), (0.0, 0), (180.0, oracle.Q_ANGLE)]:
        a = math.radians(ang)
        om = _one_kf_map([dict(u=200.0, v=200.0, desc=BASE)],
                         [_mp(pos=(0, 0, z), dmax=2.0, normal=(math.sin(a), 0, math.cos(a)))])
        assert om.query(0, tm.IDENT, 0, prm)["status"] == st, ang


def test_query_bad_and_already_found():
    om = _one_kf_map([dict(u=250.0, v=250.0, desc=BASE, mp=0)], [_mp(), _mp(flags=1)])
    assert om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))["status"] == oracle.Q_FOUND
    assert om.query(0, tm.IDENT, 1, (4, 50, 0, 0, 0))["status"] == oracle.Q_BAD


def test_window_is_strict_square_and_level_filter():
    # level 0 predicted, r = 4 exactly: |du| < 4 and |dv| < 4, octave in [-1, 0]
    feats = [dict(u=254.0, v=250.0, desc=BASE),            # |du| = r  -> out (strict)
             dict(u=253.99, v=250.0, desc=BASE),           # in
             dict(u=246.01, v=253.99, desc=BASE),          # in (square, not disc)
             dict(u=250.0, v=245.99, desc=BASE),           # out
             dict(u=250.0, v=250.0, desc=BASE, oct=1)]     # octave 1 > predicted 0 -> out
    om = _one_kf_map(feats, [_mp()])
    r = om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))
    assert r["ncand"] == 2 and r["best_f"] == 1
    # predicted level 2 (d * 1.2^2 >= dmax > d * 1.2): octaves 1 and 2 are candidates
    dmax = D0 * 1.2 ** 1.5
    feats = [dict(u=250.0, v=250.0, desc=BASE, oct=o) for o in range(5)]
    om = _one_kf_map(feats, [_mp(dmax=dmax)])
    r = om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))
    assert r["level"] == 2 and r["radius"] == 4.0 * 1.2 * 1.2
    assert r["ncand"] == 2 and r["best_f"] == 1


def test_best_second_and_tie_break_by_feature_index():
    hs = [20, 10, 12, 10, 30]
    feats = [dict(u=250.0, v=250.0, desc=tm.desc_with_h(BASE, h, offset=7 * i)) for i, h in enumerate(hs)]
    om = _one_kf_map(feats, [_mp()])
    r = om.query(0, tm.IDENT, 0, (4, 50, 0, 0, 0))
    assert (r["best_f"], r["best_h"], r["second_h"], r["ncand"]) == (1, 10, 10, 5)


def test_brute_force_all_pairs_minima():
    """All features in the window at the predicted octave: the oracle's per-query
    best/second equal the minima of the full Hamming matrix (numpy unpackbits)."""
    rng = np.random.default_rng(8)
    nf, nq = 40, 25
    fdesc = rng.integers(0, 256, (nf, 32), dtype=np.uint8)
    qdesc = rng.integers(0, 256, (nq, 32), dtype=np.uint8)
    qdesc[3] = fdesc[7]
    qdesc[4] = fdesc[2]
    fdesc[9] = fdesc[2]                                   # a tie: lower index must win
    feats = [dict(u=float(rng.uniform(150, 350)), v=float(rng.uniform(150, 350)), desc=fdesc[i])
             for i in range(nf)]
    mps = [_mp(desc=qdesc[j], dmax=1.1) for j in range(nq)]
    om = _one_kf_map(feats, mps)
    Hm = np.unpackbits(qdesc[:, None, :] ^ fdesc[None, :, :], axis=2).sum(axis=2)
    for j in range(nq):
        r = om.query(0, tm.IDENT, j, (1000, 256, 0, 0, 0))
        srt = np.sort(Hm[j])
        assert r["ncand"] == nf
        assert r["best_h"] == srt[0] and r["best_f"] == int(np.argmin(Hm[j]))
        assert r["second_h"] == srt[1]
    assert om.query(0, tm.IDENT, 4, (1000, 256, 0, 0, 0))["best_f"] == 2


def test_ratio_golden_cases():
    g = json.load(open(os.path.join(GOLD, "ratio_cases.json")))
    num, den = g["ratio"]
    for c in g["cases"]:
        feats = [dict(u=250.0, v=250.0, desc=tm.desc_with_h(BASE, c["best"])),
                 dict(u=250.0, v=250.0, desc=tm.desc_with_h(BASE, c["second"], offset=100))]
        om = _one_kf_map(feats, [_mp()])
        out = om.fuse([0], [0], (4, 100, num, den, 0), window_S=tm.IDENT[None])
        assert out["counts"]["proposals"] == int(c["kept"]), c
        assert out["counts"]["ratio_rej"] == int(not c["kept"]), c


# ------------------------------------------------------------ fusion (O7-O9)
def test_two_mps_one_feature_lower_index_wins():
    feats = [dict(u=250.0, v=250.0, desc=BASE)]
    d10a = tm.desc_with_h(BASE, 10)
    d10b = tm.desc_with_h(BASE, 10, offset=50)
    om = _one_kf_map(feats, [_mp(desc=d10b), _mp(desc=d10a), _mp(desc=tm.desc_with_h(BASE, 9), flags=1)])
    out = om.fuse([0], [0, 1, 2], (4, 50, 0, 0, 0), window_S=tm.IDENT[None])
    assert out["winner"][0] == (10 << 32) | 0
    assert om.feat_mp[0] == 0 and out["counts"]["added"] == 1


def test_constructed_duplicate_loop_point_survives():
    # KF0 (window) holds MP 2 in slot 0; loop MP 0 matches slot 0 (H=5); KF1 also observes MP 2.
    kf0 = dict(feats=[dict(u=250.0, v=250.0, desc=BASE, mp=2), dict(u=100.0, v=100.0, desc=~BASE)])
    kf1 = dict(feats=[dict(u=10.0, v=10.0, desc=BASE, mp=2), dict(u=300.0, v=300.0, desc=BASE, mp=0)])
    mps = [_mp(desc=tm.desc_with_h(BASE, 5)), _mp(pos=(0.5, 0.5, -1.0)), _mp(desc=BASE)]
    om = oracle.OracleMap(arrays=tm.build([kf0, kf1], mps), cams=[tm.PIN])
    out = om.fuse([0], [0, 1], (4, 50, 0, 0, 0), window_S=tm.IDENT[None])
    c = out["counts"]
    assert c["victims"] == 1 and c["victim_prop"] == 1
    assert out["victim"][2] == (5 << 32) | 0
    assert om.feat_mp.tolist() == [0, -1, -1, 0]       # KF1: rewired slot duplicates slot 1 -> cleared
    assert om.mp_flags[2] & 1 and om.mp_replaced_by[2] == 0
    assert om.mp_nobs.tolist() == [2, 0, 0]
    assert c["rewired"] == 2 and c["dup_cleared"] == 1


def test_disjoint_loop_points_change_nothing():
    feats = [dict(u=250.0, v=250.0, desc=BASE, mp=1)]
    om = _one_kf_map(feats, [_mp(pos=(0.5, 0.5, -1.0)), _mp()])
    before = om.feat_mp.copy()
    out = om.fuse([0], [0], (4, 50, 0, 0, 0), window_S=tm.IDENT[None])
    assert out["counts"]["proposals"] == 0 and np.all(om.feat_mp == before)
    assert not np.any(om.mp_flags & 1)


def test_orientation_filter_three_maxima():
    # 20 MPs, each projecting onto its own feature; rotations: 15 x 0deg, 4 x 90deg, 1 x 180deg
    rng = np.random.default_rng(9)
    feats, mps = [], []
    rots = [0.0] * 15 + [90.0] * 4 + [180.0]
    for j, rot in enumerate(rots):
        u = 100.0 + 10.0 * j
        d = rng.integers(0, 256, 32, dtype=np.uint8)
        feats.append(dict(u=u, v=250.0, desc=d, angle=(30.0 + rot) % 360.0))
        pos = ((u - 200.0) / 100.0, 0.5, 1.0)
        mps.append(_mp(pos=pos, desc=d, dmax=float(np.linalg.norm(pos)), angle=30.0))
    om = _one_kf_map(feats, mps)
    out = om.fuse([0], list(range(20)), (4, 50, 0, 0, 1), window_S=tm.IDENT[None])
    assert out["counts"]["winners"] == 20 and out["counts"]["orient_rej"] == 1
    assert out["action"][19] == 4 and om.feat_mp[19] == -1 and om.feat_mp[0] == 0
    om2 = _one_kf_map(feats[:15], mps[:15])
    out2 = om2.fuse([0], list(range(15)), (4, 50, 0, 0, 1), window_S=tm.IDENT[None])
    assert out2["counts"]["orient_rej"] == 0 and out2["counts"]["added"] == 15


def _audit(om, out, w):
    """Post-apply map consistency (SPEC.md:198, SPEC.md:420-423 as adapted)."""
    fb = om.kf_feat_begin
    for k in range(om.n_kf):
        s = om.feat_mp[fb[k]:fb[k + 1]]
        s = s[s >= 0]
        assert len(np.unique(s)) == len(s), f"KF {k} holds an MP in two slots"
    recount = np.bincount(om.feat_mp[om.feat_mp >= 0], minlength=om.n_mp)
    assert np.array_equal(recount, om.mp_nobs)
    vict = np.nonzero(out["victim"] != oracle.NONE64)[0]
    assert np.all(om.mp_nobs[vict] == 0)
    surv = om.mp_replaced_by[vict]
    assert np.all(surv >= 0) and not np.any(np.isin(surv, vict)), "chain"
    loopset = np.zeros(om.n_mp, bool)
    loopset[w.mp_list] = True
    assert np.all(loopset[surv])


@pytest.mark.parametrize("name", ["C1", "T1", "T2", "T5"])
@pytest.mark.parametrize("checks", [False, True])
def test_synthetic_ground_truth_and_audit(name, checks):
    from lcsynth import make_world
    from lcsynth.world import FUSE_PARAMS, FUSE_PARAMS_CHECKS
    w = make_world(name, 0)
    om = oracle.OracleMap(w)
    om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    prm = FUSE_PARAMS_CHECKS if checks else FUSE_PARAMS
    out = om.fuse(w.window, w.mp_list, prm, window_S=w.win_S, win_list_begin=w.win_list_begin)
    _audit(om, out, w)
    v = np.nonzero(out["victim"] != oracle.NONE64)[0]
    surv = (out["victim"][v] & 0xFFFFFFFF).astype(np.int64)
    assert len(v) > 20
    # descriptor+geometry fusion merges the same physical landmark (twins allowed to differ)
    assert np.mean(w.mp_lm[v] == w.mp_lm[surv]) >= 0.9
    added = np.nonzero(out["action"] == 1)[0]
    assert len(added) > 5


# ---------------------------------------------------------------- O3 / O10
def test_window_correction_owner_invariant_and_relative_poses():
    from lcsynth import make_world
    w = make_world("T1", 0)
    om = oracle.OracleMap(w)
    T_old = om.kf_pose.copy()
    S_corr, cnt = om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    assert cnt["corr_kf"] == len(w.window)
    ref = tm.to_mat4(oracle.sim3_compose(oracle.sim3_inverse(w.S_cw_corr), T_old[w.cur_kf]))
    for i, k in enumerate(w.window):
        M = tm.to_mat4(oracle.sim3_compose(oracle.sim3_inverse(S_corr[i]), T_old[k]))
        np.testing.assert_allclose(M, ref, atol=1e-12 * max(1.0, np.abs(ref).max()))
        # independent: S_iw^corr = T_iw T_wc S_cw^corr via 4x4 products
        np.testing.assert_allclose(tm.to_mat4(S_corr[i]),
                                   tm.to_mat4(T_old[k]) @ np.linalg.inv(tm.to_mat4(T_old[w.cur_kf]))
                                   @ tm.to_mat4(w.S_cw_corr), atol=1e-9)
        assert om.kf_pose[k][12] == 1.0


def test_window_correction_identity_translation_scale():
    from lcsynth import make_world
    w = make_world("T1", 0)
    c = w.cur_kf
    # identity: S_cw^corr = T_cw -> poses and points unchanged
    om = oracle.OracleMap(w)
    om.correct_window(c, om.kf_pose[c].copy(), w.window)
    np.testing.assert_allclose(om.kf_pose, w.kf_pose, atol=1e-12)
    np.testing.assert_allclose(om.mp_pos, w.mp_pos, rtol=2e-7, atol=1e-7)
    # pure translation t0 in the world: relative window poses preserved, points shift by -t0
    t0 = np.array([1.0, 0.0, 0.0])
    Tr = tm.IDENT.copy()
    Tr[9:12] = t0
    om = oracle.OracleMap(w)
    om.correct_window(c, oracle.sim3_compose(w.kf_pose[c], Tr), w.window)
    for k in w.window:
        rel_new = tm.to_mat4(om.kf_pose[k]) @ np.linalg.inv(tm.to_mat4(om.kf_pose[c]))
        rel_old = tm.to_mat4(w.kf_pose[k]) @ np.linalg.inv(tm.to_mat4(w.kf_pose[c]))
        np.testing.assert_allclose(rel_new, rel_old, atol=1e-9)
    moved = om.mp_corr_ref >= 0
    assert moved.sum() > 10
    np.testing.assert_allclose(om.mp_pos[moved], w.mp_pos[moved] - t0, atol=1e-5)
    # scale: S_cw^corr = 0.5 * T_cw (scaled about the current camera) -> distances of the
    # corrected points to the current camera centre double, whichever window KF owns them
    Sh = tm.IDENT.copy()
    Sh[12] = 0.5
    om = oracle.OracleMap(w)
    om.correct_window(c, oracle.sim3_compose(Sh, w.kf_pose[c]), w.window)
    for q in np.nonzero(om.mp_corr_ref >= 0)[0][:200]:
        R, t = w.kf_pose[c][:9].reshape(3, 3), w.kf_pose[c][9:12]
        cen = -R.T @ t
        d0 = np.linalg.norm(w.mp_pos[q].astype(np.float64) - cen)
        d1 = np.linalg.norm(om.mp_pos[q].astype(np.float64) - cen)
        assert abs(d1 / d0 - 2.0) < 1e-5


def test_all_propagation_identity_and_scale():
    from lcsynth import make_world
    w = make_world("T1", 0)
    om = oracle.OracleMap(w)
    om.correct_all(w.kf_pose.copy())
    np.testing.assert_allclose(om.kf_pose, w.kf_pose, atol=0)
    np.testing.assert_allclose(om.mp_pos, w.mp_pos, rtol=2e-7, atol=1e-7)
    Sh = tm.IDENT.copy()
    Sh[12] = 0.5
    om = oracle.OracleMap(w)
    cnt = om.correct_all(np.stack([oracle.sim3_compose(Sh, T) for T in w.kf_pose]))
    good = (w.mp_flags & 1) == 0
    assert cnt["corr_mp"] == good.sum()
    for q in np.nonzero(good)[0][:300]:
        k = w.mp_ref_kf[q]
        R, t = w.kf_pose[k][:9].reshape(3, 3), w.kf_pose[k][9:12]
        cen = -R.T @ t
        d0 = np.linalg.norm(w.mp_pos[q].astype(np.float64) - cen)
        d1 = np.linalg.norm(om.mp_pos[q].astype(np.float64) - cen)
        assert abs(d1 / d0 - 2.0) < 1e-5
    bad = np.nonzero(~good)[0]
    assert np.array_equal(om.mp_pos[bad], w.mp_pos[bad])


def test_all_after_window_uses_corrected_reference():
    """O10 after O3: window MPs use S^pre = S^corr of their owner; with S^opt = S^pre
    the corrected points stay put."""
    from lcsynth import make_world
    w = make_world("T1", 0)
    om = oracle.OracleMap(w)
    S_corr, _ = om.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    pos_after_window = om.mp_pos.copy()
    S_opt = om.kf_pose.copy()
    for i, k in enumerate(w.window):
        S_opt[k] = S_corr[i]
    om.correct_all(S_opt)
    np.testing.assert_allclose(om.mp_pos, pos_after_window, rtol=2e-7, atol=2e-7)


# -------------------------------------------------------------------- SBP
def test_sbp_taken_features_and_points():
    feats = [dict(u=250.0, v=250.0, desc=BASE), dict(u=251.0, v=250.0, desc=tm.desc_with_h(BASE, 3))]
    om = _one_kf_map(feats, [_mp(), _mp(desc=tm.desc_with_h(BASE, 1))])
    prm = [(4, 50, 0, 0, 0)]
    r = om.search_by_projection([0], tm.IDENT[None], [0], prm, [0, 2], [0, 1])
    assert r["feat_mp"].tolist() == [0, -1] and r["feat_dist"].tolist() == [0, -1]
    # feature 0 taken by MP 1: MP 1 is skipped, MP 0 falls to feature 1
    r = om.search_by_projection([0], tm.IDENT[None], [0], prm, [0, 2], [0, 1], pair_taken=[1, -1])
    assert r["feat_mp"].tolist() == [1, 0] and r["feat_dist"].tolist() == [-1, 3]
    assert r["counts"][0][oracle.COUNTER_NAMES.index("skip_found")] == 1


# ----------------------------------------------------------------------------
# O11 map-point refresh (readings A33-A37)
# ----------------------------------------------------------------------------
def _pose_at(O):
    """SE3 world->camera pose with identity rotation and camera centre O."""
    S = tm.IDENT.copy()
    S[9:12] = -np.asarray(O, np.float64)
    return S


def _refresh_map(descs, centres, octs, pos, ref_kf=0, flags=0, extra_feats=0):
    """One map point observed once by each of len(descs) keyframes (centres[i],
    octave octs[i]), plus optional unassociated clutter features."""
    base = tm.desc_from_bits([])
    kfs = []
    for i, d in enumerate(descs):
        feats = [dict(u=1.0, v=1.0, desc=base) for _ in range(extra_feats)]
        feats.append(dict(u=10.0, v=10.0, oct=int(octs[i]), desc=d, mp=0))
        kfs.append(dict(pose=_pose_at(centres[i]), feats=feats))
    mps = [dict(pos=tuple(pos), desc=base, normal=(0.0, 0.0, 1.0), dmax=1.0, ref_kf=ref_kf, flags=flags)]
    return oracle.OracleMap(arrays=tm.build(kfs, mps), cams=[tm.PIN])


def test_refresh_descriptor_special_cases():
    rng = np.random.default_rng(11)
    d = [rng.integers(0, 256, 32, dtype=np.uint8) for _ in range(3)]
    # N = 1: the only observation
    om = _refresh_map(d[:1], [(0, 0, -5)], [0], (0, 0, 0))
    om.refresh(what=1)
    assert np.array_equal(om.mp_desc[0], d[0])
    # N = 2: both medians are 0 (sorted row [0, h], index floor(1/2) = 0) -> the first
    om = _refresh_map(d[:2], [(0, 0, -5), (1, 0, -5)], [0, 0], (0, 0, 0))
    om.refresh(what=1)
    assert np.array_equal(om.mp_desc[0], d[0])
    # N = 3: A, B = A^1 bit, C = A^100 bits -> medians 1, 1, 99 -> A (first of the tie)
    A = d[0]
    B = tm.desc_with_h(A, 1, offset=200)
    Cd = tm.desc_with_h(A, 100, offset=0)
    om = _refresh_map([Cd, A, B], [(0, 0, -5), (1, 0, -5), (2, 0, -5)], [0, 0, 0], (0, 0, 0))
    om.refresh(what=1)
    assert np.array_equal(om.mp_desc[0], A)


def test_refresh_descriptor_planted_medoid():
    """Disjoint bit flips around a centre: d(i, j) = w_i + w_j (i != j). With the weights
    sorted a_1 < a_2 < ... and m = floor((N-1)/2), the k-th smallest has median
    a_k + a_m (k > m) or a_k + a_{m+1} (k <= m): the minimum a_1 + a_{m+1} is unique for
    N >= 5 and shared by a_1 and a_2 for N in {3, 4} (then the earlier observation)."""
    rng = np.random.default_rng(12)
    for trial in range(20):
        N = int(rng.integers(3, 12))
        w = rng.permutation(np.arange(1, 60))[:N]
        centre = rng.integers(0, 256, 32, dtype=np.uint8)
        descs, off = [], 0
        for wi in w:
            descs.append(tm.desc_with_h(centre, int(wi), offset=off))
            off += int(wi)
        if off > 256:
            continue
        om = _refresh_map(descs, [(i, 0, -5) for i in range(N)], [0] * N, (0, 0, 0))
        om.refresh(what=1)
        order = np.argsort(w)
        exp = int(order[0]) if N >= 5 else int(min(order[0], order[1]))
        assert np.array_equal(om.mp_desc[0], descs[exp]), (trial, w)


def test_refresh_normal_and_depth_closed_forms():
    d = [tm.desc_from_bits([i]) for i in range(4)]
    # cameras along +x and +y of the point: unit vectors (-1,0,0), (0,-1,0) -> mean (-0.5,-0.5,0)
    om = _refresh_map(d[:2], [(4, 0, 0), (0, 3, 0)], [2, 0], (0, 0, 0), ref_kf=0)
    om.refresh(what=2)
    assert np.array_equal(om.mp_normal[0], np.float32([-0.5, -0.5, 0.0]))
    # dmax = |p - O_ref| * 1.2^octave(ref observation) = 4 * 1.44
    assert om.mp_max_dist[0] == np.float32(4.0 * 1.2 * 1.2)
    # symmetric cameras: the unit vectors cancel
    om = _refresh_map(d[:2], [(2, 0, 0), (-7, 0, 0)], [0, 0], (0, 0, 0), ref_kf=1)
    om.refresh(what=2)
    assert np.array_equal(om.mp_normal[0], np.float32([0, 0, 0]))
    assert om.mp_max_dist[0] == np.float32(7.0)
    # translation invariance: moving point and cameras together changes nothing
    om2 = _refresh_map(d[:3], [(1, 2, 3), (4, -1, 0), (0, 0, 9)], [1, 3, 0], (0.5, 0.25, 0.125), ref_kf=2)
    om3 = _refresh_map(d[:3], [(11, 12, 13), (14, 9, 10), (10, 10, 19)], [1, 3, 0], (10.5, 10.25, 10.125),
                       ref_kf=2)
    om2.refresh(what=2)
    om3.refresh(what=2)
    assert np.allclose(om2.mp_normal, om3.mp_normal, atol=1e-6)
    assert abs(om2.mp_max_dist[0] - om3.mp_max_dist[0]) < 1e-5
    # the normal is the mean of unit vectors: its norm is <= 1, == 1 iff all agree
    assert np.linalg.norm(om2.mp_normal[0]) < 1.0
    om4 = _refresh_map(d[:3], [(0, 0, -1), (0, 0, -2), (0, 0, -8)], [0, 0, 0], (0, 0, 0))
    om4.refresh(what=2)
    assert np.array_equal(om4.mp_normal[0], np.float32([0, 0, 1]))


def test_refresh_skips_bad_unobserved_and_foreign_ref():
    d = [tm.desc_from_bits([i]) for i in range(2)]
    om = _refresh_map(d, [(4, 0, 0), (0, 3, 0)], [0, 0], (0, 0, 0), flags=1)
    before = (om.mp_desc.copy(), om.mp_normal.copy(), om.mp_max_dist.copy())
    c = om.refresh(what=3)
    assert c["refresh_mp"] == 0
    assert np.array_equal(om.mp_desc, before[0]) and np.array_equal(om.mp_normal, before[1])
    # reference keyframe that does not observe the point: depth range unchanged
    om = _refresh_map(d, [(4, 0, 0), (0, 3, 0)], [0, 0], (0, 0, 0), ref_kf=5)
    om.refresh(what=2)
    assert om.mp_max_dist[0] == np.float32(1.0)
    # an index list selects the points; counters count points and observations
    om = _refresh_map(d, [(4, 0, 0), (0, 3, 0)], [0, 0], (0, 0, 0), extra_feats=3)
    c = om.refresh(mp_idx=[0], what=3)
    assert c["refresh_mp"] == 1 and c["refresh_obs"] == 2


# ----------------------------------------------------------------------------
# O12 covisibility recount (SPEC.md update_connections examples;
# DESIGN.md readings A38-A40)
# ----------------------------------------------------------------------------
def _conn_map(holdings, bad=()):
    """holdings[k] = list of map-point ids held by keyframe k (one slot each)."""
    n_mp = max([q for h in holdings for q in h] + [0]) + 1
    base = tm.desc_from_bits([])
    kfs = [dict(feats=[dict(u=1.0 + i, v=1.0, desc=base, mp=int(q)) for i, q in enumerate(h)] or
                [dict(u=1.0, v=1.0, desc=base)]) for h in holdings]
    mps = [dict(pos=(0.0, 0.0, 1.0), desc=base, flags=1 if q in bad else 0) for q in range(n_mp)]
    return oracle.OracleMap(arrays=tm.build(kfs, mps), cams=[tm.PIN])


def test_connections_spec_examples():
    # "keyframe sharing 20 points with kf A and 5 with kf B -> weights {A:20, B:5}"
    om = _conn_map([list(range(30)), list(range(20)) + [40, 41], list(range(25, 30))])
    n, kf, w, c = om.update_connections([0], th=5)
    assert n[0] == 2 and list(kf[0, :2]) == [1, 2] and list(w[0, :2]) == [20, 5]
    n, kf, w, c = om.update_connections([0], th=15)    # B below the threshold: dropped
    assert n[0] == 1 and kf[0, 0] == 1 and w[0, 0] == 20
    # "keyframe whose every weight < 15 -> retains exactly one edge (max, tie -> lowest id)"
    om = _conn_map([list(range(10)), list(range(7)), list(range(3, 10)), [0]])
    n, kf, w, c = om.update_connections([0], th=15)
    assert n[0] == 1 and kf[0, 0] == 1 and w[0, 0] == 7
    # no shared points at all: no edge
    om = _conn_map([[0, 1], [2, 3]])
    n, kf, w, c = om.update_connections(None, th=15)
    assert list(n) == [0, 0] and c["conn_kf"] == 2 and c["conn_edges"] == 0


def test_connections_order_bad_points_and_duplicates():
    # equal weights: ascending keyframe id; larger weight first
    om = _conn_map([list(range(40)), list(range(16)), list(range(20, 40)), list(range(16)), [0, 1]])
    n, kf, w, c = om.update_connections([0], th=15)
    assert n[0] == 3 and list(kf[0, :3]) == [2, 1, 3] and list(w[0, :3]) == [20, 16, 16]
    # bad points do not count; a keyframe holding a point twice counts it once
    om = _conn_map([list(range(20)), list(range(20)) + [3], list(range(20))], bad=(0, 1))
    n, kf, w, c = om.update_connections(None, th=15)
    assert list(w[0, :2]) == [18, 18] and list(kf[0, :2]) == [1, 2]
    assert w[1, 0] == 18 and w[2, 0] == 18


def test_connections_symmetric_and_truncated():
    rng = np.random.default_rng(3)
    holdings = [sorted(rng.choice(300, size=int(rng.integers(20, 120)), replace=False).tolist())
                for _ in range(12)]
    om = _conn_map(holdings)
    n, kf, w, c = om.update_connections(None, th=1, max_edges=16)
    W = np.zeros((12, 12), np.int64)
    for a in range(12):
        for e in range(min(n[a], 16)):
            W[a, kf[a, e]] = w[a, e]
    # with th = 1 every shared keyframe is an edge; the weight matrix is symmetric and
    # equals the size of the intersection of the held sets
    for a in range(12):
        for b in range(12):
            if a != b:
                assert W[a, b] == len(set(holdings[a]) & set(holdings[b])) or n[a] > 16
    assert np.array_equal(W, W.T)
    n2, kf2, w2, _ = om.update_connections(None, th=1, max_edges=3)   # truncated rows
    assert np.array_equal(n2, n) and np.array_equal(kf2[:, :3], kf[:, :3])


# ----------------------------------------------------------------------------
# O13 Sim3 RANSAC (SPEC.md estimate_sim3_ransac examples;
# DESIGN.md readings A41-A44)
# ----------------------------------------------------------------------------
def _sim3_yaw(s, yaw_deg, t):
    a = np.deg2rad(yaw_deg)
    R = np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1.0]])
    return np.r_[R.reshape(-1), np.asarray(t, np.float64), s]


def test_jacobi4_matches_library_eigh():
    rng = np.random.default_rng(21)
    for _ in range(200):
        A = rng.standard_normal((4, 4))
        A = A + A.T
        ev, V = oracle.jacobi4(A)
        ref = np.linalg.eigh(A)[0]
        assert np.allclose(np.sort(ev), ref, rtol=1e-12, atol=1e-12)
        assert np.allclose(A @ V, V * ev, atol=1e-10)            # columns are eigenvectors
        assert np.allclose(V.T @ V, np.eye(4), atol=1e-12)


def test_horn_closed_form_cases():
    rng = np.random.default_rng(22)
    P = rng.uniform(-2, 2, (50, 3)) + [0, 0, 5]
    S = oracle.horn(P, P)                                          # identity
    assert np.allclose(S, tm.IDENT, atol=1e-12)
    T = _sim3_yaw(1.3, 10.0, (1, 2, 3))                            # SPEC: s=1.3, 10° yaw, t=(1,2,3)
    P1 = np.array([oracle.sim3_apply(T, p) for p in P])
    for n in (3, 50):
        S = oracle.horn(P1[:n], P[:n])
        assert np.allclose(S, T, atol=1e-9), (n, S - T)
    T1 = _sim3_yaw(1.0, -35.0, (0.5, -1, 2))                       # rigid: fixed scale exact
    P1 = np.array([oracle.sim3_apply(T1, p) for p in P])
    assert np.allclose(oracle.horn(P1, P, fix_scale=True), T1, atol=1e-9)


def _ransac_scene(rng, n=60, out_frac=0.3, T=None):
    T = _sim3_yaw(1.3, 10.0, (0.3, -0.2, 0.1)) if T is None else T
    Ti = oracle.sim3_inverse(T)
    P1 = rng.uniform([-2, -2, 3], [2, 2, 8], (n, 3))               # camera-1 frame
    P2 = np.array([oracle.sim3_apply(Ti, p) for p in P1])          # camera-2 frame
    inl = np.ones(n, bool)
    out = rng.choice(n, int(out_frac * n), replace=False)
    inl[out] = False
    P2[out] = rng.uniform([-2, -2, 3], [2, 2, 8], (len(out), 3))   # wrong partner
    uv1 = np.array([oracle.project(tm.PIN, p) for p in P1])
    uv2 = np.array([oracle.project(tm.PIN, p) for p in np.array([oracle.sim3_apply(Ti, p) for p in P1])])
    return T, P1, P2, uv1.astype(np.float32), uv2.astype(np.float32), inl


def _empty_map():
    base = tm.desc_from_bits([])
    return oracle.OracleMap(arrays=tm.build([dict(feats=[dict(u=1.0, v=1.0, desc=base)])],
                                            [dict(pos=(0, 0, 1), desc=base)]), cams=[tm.PIN])


def test_ransac_recovers_planted_model_and_inliers():
    rng = np.random.default_rng(23)
    om = _empty_map()
    T, P1, P2, uv1, uv2, inl = _ransac_scene(rng)
    n = len(P1)
    samples = np.array([rng.choice(n, 3, replace=False) for _ in range(200)], np.int32)
    S, ninl, mask, c = om.sim3_ransac([0, n], P1, P2, uv1, uv2, np.ones(n), np.ones(n), [0], [0],
                                      samples[None], chi2=9.210)
    assert np.array_equal(mask.astype(bool), inl)                  # exactly the constructed inliers
    assert ninl[0] == inl.sum() and c["ransac_hyp"] == 200
    assert np.allclose(S[0], T, atol=1e-6)
    # outlier-free: every sample is exact, the first one wins
    T, P1, P2, uv1, uv2, inl = _ransac_scene(rng, n=20, out_frac=0.0)
    S, ninl, mask, c = om.sim3_ransac([0, 20], P1, P2, uv1, uv2, np.ones(20), np.ones(20), [0], [0],
                                      np.array([[[0, 1, 2], [3, 4, 5]]], np.int32), refit=False)
    assert ninl[0] == 20 and np.allclose(S[0], T, atol=1e-9)


def test_ransac_degenerate_samples_and_batches():
    rng = np.random.default_rng(24)
    om = _empty_map()
    T, P1, P2, uv1, uv2, inl = _ransac_scene(rng, n=12)
    S, ninl, mask, c = om.sim3_ransac([0, 12], P1, P2, uv1, uv2, np.ones(12), np.ones(12), [0], [0],
                                      np.array([[[1, 1, 2], [4, 5, 5]]], np.int32))
    assert ninl[0] == 0 and c["ransac_hyp"] == 0 and not mask.any()   # A41: skipped
    # two problems in one batch: each solved independently
    T2, Q1, Q2, w1, w2, inl2 = _ransac_scene(rng, n=30, T=_sim3_yaw(0.8, -20.0, (1, 0, 0)))
    smp = np.array([[rng.choice(12, 3, replace=False) for _ in range(50)],
                    [rng.choice(30, 3, replace=False) for _ in range(50)]], np.int32)
    S, ninl, mask, c = om.sim3_ransac([0, 12, 42], np.r_[P1, Q1], np.r_[P2, Q2], np.r_[uv1, w1],
                                      np.r_[uv2, w2], np.ones(42), np.ones(42), [0, 0], [0, 0], smp)
    assert np.array_equal(mask.astype(bool), np.r_[inl, inl2])
    assert np.allclose(S[1], T2, atol=1e-6)


# ----------------------------------------------------------------------------
# O14 Sim3 refinement (SPEC.md refine_sim3; readings A45-A48)
# ----------------------------------------------------------------------------
def test_retraction_closed_forms():
    rng = np.random.default_rng(41)
    S = tm.random_sim3(rng)
    assert np.array_equal(oracle.sim3_retract(np.zeros(7), S), oracle.sim3_compose(tm.IDENT, S))
    for _ in range(50):
        w = rng.normal(0, 0.5, 3)
        d = np.r_[w, rng.normal(0, 1, 3), rng.uniform(-0.5, 0.5)]
        D = oracle.sim3_retract(d, tm.IDENT)
        R = D[:9].reshape(3, 3)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-14) and np.linalg.det(R) > 0
        ang = np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1))     # Cayley: angle = 2 atan |w|
        assert abs(ang - 2 * np.arctan(np.linalg.norm(w))) < 1e-12
        assert np.allclose(R @ w, w, atol=1e-14)                     # about the axis w
        assert np.allclose(D[9:12], d[3:6]) and D[12] == 1.0 + d[6]


def test_refine_fixed_point_convergence_and_outliers():
    rng = np.random.default_rng(42)
    om = _empty_map()
    T, P1, P2, uv1, uv2, inl = _ransac_scene(rng, n=80, out_frac=0.0)
    ones = np.ones(80)
    S, ninl, mask, c = om.sim3_refine([0, 80], P1, P2, uv1, uv2, ones, ones, [0], [0], T[None])
    # the truth is a fixed point up to the fp32 rounding of the keypoints (~1e-7)
    assert np.allclose(S[0], T, atol=1e-6) and ninl[0] == 80
    S0 = oracle.sim3_retract(np.r_[0.01, -0.02, 0.005, 0.05, -0.03, 0.02, 0.02], T)
    S, ninl, mask, c = om.sim3_refine([0, 80], P1, P2, uv1, uv2, ones, ones, [0], [0], S0[None], max_iter=30)
    assert np.allclose(S[0], T, atol=1e-6) and ninl[0] == 80 and c["refine_iters"] >= 2
    # 25% far outliers: Huber keeps the estimate at the truth, the mask is the planted one
    T, P1, P2, uv1, uv2, inl = _ransac_scene(rng, n=80, out_frac=0.25)
    S0 = oracle.sim3_retract(np.r_[0.005, 0.0, -0.005, 0.02, 0.0, 0.01, 0.01], T)
    S, ninl, mask, c = om.sim3_refine([0, 80], P1, P2, uv1, uv2, ones, ones, [0], [0], S0[None], max_iter=30)
    assert np.allclose(S[0], T, atol=1e-5), S[0] - T
    assert np.array_equal(mask.astype(bool), inl)
