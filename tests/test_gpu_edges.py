"""Adversarial boundary cases for the GPU's filtered (fp32 + exact fallback) predicates.

Map points and keypoints are placed so that projections land within 1e-7..1e-2 px of
the image bounds and of the square-window edges, distances sit at the distance-range
and level thresholds, and view angles at the 0.5 cosine; the GPU's decisions must equal
the oracle's fp64 decisions exactly (reading A32: no ambiguity for pinhole cameras).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from tests import tinymap as tm  # noqa: E402

rng = np.random.default_rng(77)
DELTAS = [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 5e-4, 1e-3, 3e-3, 1e-2, 3e-2]


def _rand_pose(far=0.0):
    S = tm.random_sim3(rng, scale=False)
    S[9:12] += far
    return S


def _pt_at_pixel(S, cam, u, v, z):
    """World point whose camera coordinates are ((u-cx) z / fx, (v-cy) z / fy, z)."""
    R = S[:9].reshape(3, 3)
    pc = np.array([(u - cam["cx"]) * z / cam["fx"], (v - cam["cy"]) * z / cam["fy"], z])
    return R.T @ (pc - S[9:12] / S[12])


def _build_case(far):
    cam = dict(model=0, fx=458.654, fy=457.296, cx=367.215, cy=248.375, k=(0, 0, 0, 0),
               min_x=0.0, max_x=752.0, min_y=0.0, max_y=480.0)
    S = _rand_pose(far)
    base = rng.integers(0, 256, 32, dtype=np.uint8)
    mps, feats = [], []
    # (a) projections straddling the image bounds
    for d in DELTAS:
        for sgn in (-1, 1):
            for (u, v) in [(0.0 + sgn * d, 240.0), (752.0 + sgn * d, 100.0), (300.0, 0.0 + sgn * d),
                           (400.0, 480.0 + sgn * d)]:
                p = _pt_at_pixel(S, cam, u, v, rng.uniform(2, 8))
                mps.append(dict(pos=tuple(p), desc=base, dmax=float(np.linalg.norm(p - (-S[:9].reshape(3, 3).T @ S[9:12])))))
    # (b) window edges: a feature at |du| = r +- delta around the projection
    centres = []
    for i in range(60):
        u, v = rng.uniform(40, 700), rng.uniform(40, 440)
        p = _pt_at_pixel(S, cam, u, v, rng.uniform(2, 8))
        centres.append(len(mps))
        mps.append(dict(pos=tuple(p), desc=tm.desc_with_h(base, i % 40, offset=i)))
    return cam, S, base, mps, centres


@pytest.mark.parametrize("far", [0.0, 300.0])
def test_filtered_predicates_match_oracle_at_edges(far):
    from paper_2603_17201_b200 import Context
    cam, S, base, mps, centres = _build_case(far)
    Ow = -S[:9].reshape(3, 3).T @ (S[9:12] / S[12])
    for m in mps:   # normals toward the camera, dmax consistent with level 0..7
        p = np.asarray(m["pos"], np.float64)
        m["normal"] = tuple((p - Ow) / np.linalg.norm(p - Ow))
        m.setdefault("dmax", float(np.linalg.norm(p - Ow)) * 1.2 ** rng.integers(0, 8))
    # first pass: exact projections / levels from the oracle (no features yet)
    arrays = tm.build([dict(pose=S, feats=[dict(u=1.0, v=1.0, desc=~base, oct=7)])], mps)
    om = oracle.OracleMap(arrays=arrays, cams=[cam])
    feats = []
    for qi in centres:
        r = om.query(0, S, qi, (4, 256, 0, 0, 0))
        if r["status"] != 0:
            continue
        lvl, rad = r["level"], r["radius"]
        for d in DELTAS:
            for sgn in (-1, 1):
                for axis in (0, 1):
                    uv = [r["u"], r["v"]]
                    uv[axis] += sgn * (rad + (d if rng.uniform() < 0.5 else -d))
                    feats.append(dict(u=float(uv[0]), v=float(uv[1]), oct=lvl, desc=tm.desc_with_h(base, int(rng.integers(0, 60)), offset=7)))
    # distance / angle / level thresholds: perturb dmax and normals of a few points
    for m in mps[::3]:
        p = np.asarray(m["pos"], np.float64)
        dd = float(np.linalg.norm(p - Ow))
        n = rng.integers(0, 8)
        m["dmax"] = float(np.float32(dd * 1.2 ** n * (1 + rng.choice([-1, 1]) * rng.choice([0, 1e-7, 1e-6, 1e-5]))))
    for m in mps[1::5]:
        p = np.asarray(m["pos"], np.float64)
        po = (p - Ow) / np.linalg.norm(p - Ow)
        ax = np.cross(po, [0.3, 0.2, 0.9]); ax /= np.linalg.norm(ax)
        ang = math.acos(0.5) + rng.choice([-1, 1]) * rng.choice([0, 1e-7, 1e-6, 1e-5])
        m["normal"] = tuple(math.cos(ang) * po + math.sin(ang) * ax)
    arrays = tm.build([dict(pose=S, feats=feats + [dict(u=1.0, v=1.0, desc=~base, oct=7)])], mps)
    lst = np.arange(len(mps), dtype=np.int32)
    om = oracle.OracleMap(arrays=arrays, cams=[cam])
    o = om.fuse([0], lst, (4, 256, 0, 0, 0), window_S=S[None], debug=True)
    ctx = Context(0)
    ctx.upload_map(arrays, [cam])
    g = ctx.fuse([0], lst, (4, 256, 0, 0, 0), window_S=S[None], debug=True)
    ctx2 = Context(0)
    ctx2.upload_map(arrays, [cam])
    g2 = ctx2.fuse([0], lst, (4, 256, 0, 0, 0), window_S=S[None])   # no debug: fast path only
    assert np.array_equal(g["best"], o["best"]), np.nonzero(g["best"] != o["best"])[0][:10]
    assert np.array_equal(g["ncand"], o["ncand"])
    assert np.array_equal(g["winner"], o["winner"]) and np.array_equal(g2["winner"], o["winner"])
    assert g["counts"] == o["counts"] and g2["counts"] == o["counts"]
    st = o["status"]
    assert (st == oracle.Q_BOUNDS).sum() > 20 and (st == 0).sum() > 20
