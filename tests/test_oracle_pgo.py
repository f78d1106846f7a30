"""Pins of oracle O15 (essential-graph Sim3 PGO; readings A49-A53)
against what the mathematics fixes, not against the oracle itself:

  * exp: scipy's matrix exponential of the 4x4 Lie-algebra matrix [[Omega + sigma I, u], [0, 0]]
    (an independent library routine), in every branch of A49 and across the branch edges;
  * log: scipy's matrix logarithm, and exp o log = id;
  * Jacobians: central finite differences (SPEC.md edge_jacobians: 1e-6 relative) and the
    hand-derived consistent-edge case J_i = Ad(M), J_j = -I;
  * LM: the single-edge closed form, zero-residual no-op, exact recovery of the truth of an
    "exact" graph (the unique optimum), gauge invariance, monotone accepted chi2, and the
    lambda-overflow stop of a singular system.
"""
import numpy as np
import pytest
import scipy.linalg as sl

import oracle
from lcsynth import make_pose_graph


def hat(w):
    return np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]], np.float64)


def exp_ref(x):
    """Sim3 exponential via scipy.linalg.expm of the 4x4 generator (S = [[sR, t], [0, 1]])."""
    G = np.zeros((4, 4))
    G[:3, :3] = hat(x[:3]) + x[6] * np.eye(3)
    G[:3, 3] = x[3:6]
    T = sl.expm(G)
    s = np.exp(x[6])
    out = np.zeros(13)
    out[:9] = (T[:3, :3] / s).reshape(-1)
    out[9:12] = T[:3, 3]
    out[12] = s
    return out


def S_to4(S):
    T = np.eye(4)
    T[:3, :3] = S[12] * S[:9].reshape(3, 3)
    T[:3, 3] = S[9:12]
    return T


def rand_x(rng, th, sg, u=1.0):
    w = rng.standard_normal(3)
    w *= th / np.linalg.norm(w)
    return np.concatenate([w, u * rng.standard_normal(3), [sg]])


REGIMES = [(0.7, 0.4), (2.5, -0.8), (0.3, 0.0), (0.3, 2e-4), (0.3, 1.5e-3), (5e-5, 0.3), (5e-5, 1e-4),
           (0.0, 0.0), (0.0, -0.5), (1.2e-4, 0.2), (9e-5, 9e-4), (1.1e-4, 1.1e-3), (1e-9, 1e-9)]


@pytest.mark.parametrize("th,sg", REGIMES)
def test_exp_matches_matrix_exponential(th, sg):
    rng = np.random.default_rng(int(th * 1e6) + int(abs(sg) * 1e6))
    for _ in range(5):
        x = rand_x(rng, th, sg)
        np.testing.assert_allclose(oracle.pgo_exp(x), exp_ref(x), rtol=0, atol=1e-12)


@pytest.mark.parametrize("th,sg", REGIMES)
def test_log_inverts_exp_and_matches_logm(th, sg):
    rng = np.random.default_rng(17 + int(th * 1e6))
    for _ in range(5):
        x = rand_x(rng, th, sg)
        S = exp_ref(x)
        np.testing.assert_allclose(oracle.pgo_log(S), x, rtol=0, atol=1e-10)
        if th > 1e-3:   # logm is accurate away from the identity
            L = np.real(sl.logm(S_to4(S)))
            ref = np.concatenate([[L[2, 1], L[0, 2], L[1, 0]], L[:3, 3], [np.trace(L[:3, :3]) / 3]])
            np.testing.assert_allclose(oracle.pgo_log(S), ref, rtol=0, atol=1e-9)


def rand_S(rng, th=1.0, sc=0.3):
    return exp_ref(rand_x(rng, th * rng.random(), sc * rng.standard_normal()))


def test_jacobians_match_central_differences():
    """SPEC.md edge_jacobians: 100 random edges, autodiff = central FD (h = 1e-6) within 1e-6 rel."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        Si, Sj = rand_S(rng), rand_S(rng)
        # a measurement near consistency, so the residual rotation stays well inside (-pi, pi)
        M = oracle.sim3_compose(exp_ref(0.3 * rng.standard_normal(7)),
                                oracle.sim3_compose(Sj, oracle.sim3_inverse(Si)))
        e, Ji, Jj = oracle.pgo_edge(M, Si, Sj)
        h = 1e-6
        for which, J in ((0, Ji), (1, Jj)):
            Jfd = np.zeros((7, 7))
            for k in range(7):
                d = np.zeros(7)
                d[k] = h
                Sp = [Si.copy(), Sj.copy()]
                Sm = [Si.copy(), Sj.copy()]
                Sp[which] = oracle.sim3_compose(exp_ref(d), Sp[which])
                Sm[which] = oracle.sim3_compose(exp_ref(-d), Sm[which])
                ep = oracle.pgo_edge(M, *Sp)[0]
                em = oracle.pgo_edge(M, *Sm)[0]
                Jfd[:, k] = (ep - em) / (2 * h)
            np.testing.assert_allclose(J, Jfd, rtol=1e-6, atol=1e-6 * max(1.0, np.abs(J).max()))


def adjoint(M):
    """Hand-derived Sim3 adjoint for the tangent order (omega, upsilon, sigma):
    M exp(x) M^-1 = exp(Ad x), Ad = [[R, 0, 0], [[t]x R, s R, -t], [0, 0, 1]]."""
    R, t, s = M[:9].reshape(3, 3), M[9:12], M[12]
    A = np.zeros((7, 7))
    A[:3, :3] = R
    A[3:6, :3] = hat(t) @ R
    A[3:6, 3:6] = s * R
    A[3:6, 6] = -t
    A[6, 6] = 1.0
    return A


def test_consistent_edge_jacobians_are_adjoint_and_minus_identity():
    """e = log(M exp(d_i) S_i S_j^-1 exp(-d_j)) with M S_i S_j^-1 = I: J_i = Ad(M), J_j = -I."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        Si, Sj = rand_S(rng), rand_S(rng)
        M = oracle.sim3_compose(Sj, oracle.sim3_inverse(Si))
        e, Ji, Jj = oracle.pgo_edge(M, Si, Sj)
        assert np.abs(e).max() < 1e-12
        np.testing.assert_allclose(Ji, adjoint(M), rtol=0, atol=1e-10)
        np.testing.assert_allclose(Jj, -np.eye(7), rtol=0, atol=1e-10)


def test_first_order_residual():
    """Consistent edge, vertex i perturbed by exp(d), |d| = 1e-6: e = Ad(M) d to first order."""
    rng = np.random.default_rng(6)
    Si, Sj = rand_S(rng), rand_S(rng)
    M = oracle.sim3_compose(Sj, oracle.sim3_inverse(Si))
    d = rng.standard_normal(7)
    d *= 1e-6 / np.linalg.norm(d)
    e = oracle.pgo_edge(M, oracle.sim3_compose(exp_ref(d), Si), Sj)[0]
    np.testing.assert_allclose(e, adjoint(M) @ d, rtol=0, atol=1e-6 * 1e-4)


def test_single_edge_closed_form():
    """Two vertices, 0 fixed, one inconsistent edge: the free vertex converges to M o S_0."""
    rng = np.random.default_rng(7)
    S0, S1 = rand_S(rng), rand_S(rng)
    M = oracle.sim3_compose(exp_ref(0.5 * rng.standard_normal(7)),
                            oracle.sim3_compose(S1, oracle.sim3_inverse(S0)))
    S, tr, (c0, c1), cnt = oracle.pgo(np.stack([S0, S1]), [1, 0], [[0, 1]], M[None], max_iter=50,
                                      eps_dx=1e-12)
    assert c0 > 1e-3 and c1 < 1e-18
    np.testing.assert_array_equal(S[0], S0)
    np.testing.assert_allclose(S[1], oracle.sim3_compose(M, S0), rtol=0, atol=1e-9)
    assert oracle.PGO_STOP[cnt["pgo_stop"]] in ("dx", "chi2")


def test_zero_residual_is_a_no_op():
    g = make_pose_graph("G0", 1, mode="exact")
    S, tr, (c0, c1), cnt = oracle.pgo(g.S_true, g.fixed, g.edges, g.M)
    assert c0 < 1e-28 or cnt["pgo_accepted"] == 0
    if c0 == 0.0:
        assert cnt["pgo_iters"] == 0 and oracle.PGO_STOP[cnt["pgo_stop"]] == "zero"
    np.testing.assert_allclose(S, g.S_true, rtol=0, atol=1e-13)


@pytest.mark.parametrize("seed", [0, 1])
def test_exact_graph_recovers_the_truth(seed):
    """All measurements from the truth, vertex 0 fixed at the truth: the unique optimum is
    the truth (chi2 = 0), reached from the drifted start."""
    g = make_pose_graph("G1", seed, mode="exact")
    S, tr, (c0, c1), cnt = oracle.pgo(g.S_init, g.fixed, g.edges, g.M, max_iter=50)
    assert c0 > 1e-3 and c1 < 1e-18
    np.testing.assert_allclose(S, g.S_true, rtol=0, atol=1e-8)
    acc = tr[tr[:, 3] == 1]
    assert np.all(acc[:, 2] < acc[:, 0])


def test_drift_graph_monotone_and_gauge_invariant():
    g = make_pose_graph("G1", 2)
    S, tr, (c0, c1), cnt = oracle.pgo(g.S_init, g.fixed, g.edges, g.M)
    assert c1 < 0.2 * c0
    acc = tr[tr[:, 3] == 1]
    assert len(acc) >= 2 and np.all(np.diff(acc[:, 2]) < 0)
    assert np.all((tr[:, 1] >= 1e-12) & (tr[:, 1] <= 1e8))
    # gauge: a global change of world frame S_v -> S_v o G leaves every residual unchanged
    G = exp_ref(np.array([0.2, -0.1, 0.3, 1.0, -2.0, 0.5, 0.3]))
    S0g = np.stack([oracle.sim3_compose(s, G) for s in g.S_init])
    Sg, trg, (c0g, c1g), _ = oracle.pgo(S0g, g.fixed, g.edges, g.M)
    np.testing.assert_allclose(c1g, c1, rtol=1e-9)
    Ginv = oracle.sim3_inverse(G)
    back = np.stack([oracle.sim3_compose(s, Ginv) for s in Sg])
    np.testing.assert_allclose(back, S, rtol=0, atol=1e-9)


def test_singular_system_stops_on_lambda():
    """A free vertex without edges makes H singular: every LDL^T fails, lambda overflows."""
    g = make_pose_graph("G0", 0)
    S0 = np.concatenate([g.S_init, g.S_init[:1]])
    fx = np.concatenate([g.fixed, [0]]).astype(np.uint8)
    S, tr, (c0, c1), cnt = oracle.pgo(S0, fx, g.edges, g.M, max_iter=100)
    assert oracle.PGO_STOP[cnt["pgo_stop"]] == "lambda"
    assert cnt["pgo_accepted"] == 0 and np.all(tr[:, 2] == -1.0)
    np.testing.assert_array_equal(S, S0)
