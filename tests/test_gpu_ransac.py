"""Batched Sim3 RANSAC (lc_sim3_ransac) against oracle O13: the
selected models (bit for bit: the same fp64 expressions, the same Jacobi order), inlier
counts, masks and counters, on planted scenes with outliers, pinhole and
Kannala-Brandt cameras, staged (<= 512) and global-memory problem sizes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from lcsynth import make_world  # noqa: E402


@pytest.fixture(scope="module")
def Ctx():
    from paper_2603_17201_b200 import Context, build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return Context


def _batch(rng, cam, n_prob=24, big=(700,)):
    sizes = [int(x) for x in rng.integers(3, 200, n_prob - len(big))] + list(big)
    P1s, P2s, U1, U2, S1, S2, smp, truth = [], [], [], [], [], [], [], []
    for n in sizes:
        a = rng.uniform(-0.6, 0.6)
        R = np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1.0]])
        T = np.r_[R.reshape(-1), rng.uniform(-0.3, 0.3, 3), rng.uniform(0.7, 1.4)]
        Ti = oracle.sim3_inverse(T)
        P1 = rng.uniform([-1.5, -1.5, 3], [1.5, 1.5, 8], (n, 3))
        P2t = np.array([oracle.sim3_apply(Ti, p) for p in P1])
        P2 = P2t.copy()
        out = rng.choice(n, int(rng.uniform(0, 0.5) * n), replace=False)
        P2[out] = rng.uniform([-1.5, -1.5, 3], [1.5, 1.5, 8], (len(out), 3))
        U1.append(np.array([oracle.project(cam, p) for p in P1], np.float32) + rng.normal(0, 0.3, (n, 2)).astype(np.float32))
        U2.append(np.array([oracle.project(cam, p) for p in P2t], np.float32))
        lv = rng.integers(0, 8, n)
        S1.append((1.2 ** (2 * lv)).astype(np.float32))
        S2.append((1.2 ** (2 * rng.integers(0, 8, n))).astype(np.float32))
        P1s.append(P1)
        P2s.append(P2)
        s = np.array([rng.choice(n, 3, replace=n < 3) for _ in range(300)], np.int32)
        rep = rng.random(300) < 0.05
        s[rep, 1] = s[rep, 0]                        # repeated index: skipped (A41)
        smp.append(s)
        truth.append(T)
    pb = np.r_[0, np.cumsum(sizes)].astype(np.int32)
    return (pb, np.concatenate(P1s), np.concatenate(P2s), np.concatenate(U1), np.concatenate(U2),
            np.concatenate(S1), np.concatenate(S2), np.stack(smp), truth)


@pytest.mark.parametrize("world", ["T1", "T2"], ids=["pinhole", "kannala-brandt"])
@pytest.mark.parametrize("refit", [True, False])
def test_ransac_batch_matches_oracle(Ctx, world, refit):
    w = make_world(world, 0)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    rng = np.random.default_rng(31)
    pb, P1, P2, U1, U2, S1, S2, smp, truth = _batch(rng, w.cam)
    n_prob = len(pb) - 1
    cams = np.zeros(n_prob, np.int32)
    smp[3, :, :] = [0, 0, 1]                         # a problem with no valid sample (A41)
    g = ctx.sim3_ransac(pb, P1, P2, U1, U2, S1, S2, cams, cams, smp, refit=refit)
    o = om.sim3_ransac(pb, P1, P2, U1, U2, S1, S2, cams, cams, smp, refit=refit)
    assert np.array_equal(g[1], o[1]), "inlier counts"
    assert np.array_equal(g[2], o[2]), "masks"
    assert np.array_equal(g[0], o[0]), "models"
    assert g[3]["ransac_hyp"] == o[3]["ransac_hyp"] and g[3]["ransac_inliers"] == o[3]["ransac_inliers"]
    assert g[1][3] == 0 and not g[0][3].any()
    good = [b for b in range(n_prob) if b != 3 and g[1][b] >= 10]
    assert len(good) > n_prob // 2


@pytest.mark.parametrize("world", ["T1", "T2"], ids=["pinhole", "kannala-brandt"])
def test_refine_batch_matches_oracle(Ctx, world):
    """Gauss-Newton Sim3 refinement (lc_sim3_refine, readings A45-A48) against oracle O14
    from the RANSAC models: pinhole is rational arithmetic -> bit-identical; the
    Kannala-Brandt projection uses atan2 (libm vs CUDA may differ by <= 2 ulp) -> models
    within 1e-9, same masks and counters."""
    w = make_world(world, 0)
    ctx = Ctx(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    om = oracle.OracleMap(w)
    rng = np.random.default_rng(32)
    pb, P1, P2, U1, U2, S1, S2, smp, truth = _batch(rng, w.cam, n_prob=16, big=(600,))
    cams = np.zeros(len(pb) - 1, np.int32)
    S0 = om.sim3_ransac(pb, P1, P2, U1, U2, S1, S2, cams, cams, smp)[0]
    ok = np.abs(S0).sum(1) > 0
    g = ctx.sim3_refine(pb, P1, P2, U1, U2, S1, S2, cams, cams, S0, max_iter=10)
    o = om.sim3_refine(pb, P1, P2, U1, U2, S1, S2, cams, cams, S0, max_iter=10)
    assert np.array_equal(g[1], o[1]) and np.array_equal(g[2], o[2])
    assert g[3]["refine_inliers"] == o[3]["refine_inliers"]
    if world == "T1":
        assert g[3]["refine_iters"] == o[3]["refine_iters"]
        assert np.array_equal(g[0][ok], o[0][ok])
    else:   # the |d|^2 < 1e-20 stop sits at the ulp level: at most one step apart per problem
        assert abs(g[3]["refine_iters"] - o[3]["refine_iters"]) <= len(pb) - 1
        assert np.allclose(g[0][ok], o[0][ok], rtol=1e-8, atol=1e-9)   # one last step (|d| < 1e-10) apart
    # the refinement does not lose inliers against the RANSAC models
    r = om.sim3_ransac(pb, P1, P2, U1, U2, S1, S2, cams, cams, smp)[1]
    assert np.all(g[1][ok] >= r[ok] - 2)
