"""Seeded synthetic essential graphs.

An essential graph as ORB-SLAM3's loop closer builds it after a loop (PAPER.md:244-248
§IV.F; SPEC.md build_essential_problem): one vertex per keyframe (world->camera Sim3),
spanning-tree edges (parent = previous keyframe, 10% the one before), covisibility
edges to the next `cov` keyframes (kept with probability 0.7, standing in for
"weight >= 100"), and loop edges between the last and the first `n_loop` keyframes.

The keyframes lie on a closed circle traversed once (camera looking along the path
with yaw/pitch jitter). Two measurement modes:

  * "drift" (the loop-closing case, default): the initial estimates are the truth
    with an accumulated odometry drift (random walk in rotation, translation and
    monocular scale); tree and covisibility measurements are taken from the drifted
    estimates (M = S_j S_i^-1, so they are consistent with them) with N(0, noise)
    perturbations; loop measurements come from the truth. The loop error is what the
    optimisation distributes along the graph.
  * "exact": every measurement comes from the truth, the initial estimates are the
    drifted ones; the optimum is the truth itself (chi2 = 0), up to the gauge fixed by
    vertex 0 (which starts at the truth).

Vertex 0 (the loop keyframe) is fixed. Everything is numpy (PCG64); no oracle or CUDA
arithmetic lives here -- the Sim3 helpers only construct inputs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .world import _compose, _inverse, _rodrigues, _to13

GRAPHS = {
    # name: (n keyframes, covisibility span, loop edges, ring radius m)
    "G0": (12, 3, 2, 2.0),
    "G1": (60, 5, 4, 4.0),
    "C2": (300, 6, 6, 10.0),      # EuRoC MH scale
    "C3": (1000, 6, 8, 25.0),     # TUM-VI room scale (C3)
    "C5": (5000, 6, 12, 80.0),    # large map (C5)
}


@dataclass
class PoseGraph:
    name: str
    S_init: np.ndarray   # [n, 13] initial world->camera Sim3 estimates
    S_true: np.ndarray   # [n, 13] ground truth
    fixed: np.ndarray    # [n] uint8
    edges: np.ndarray    # [m, 2] int32 (i, j)
    M: np.ndarray        # [m, 13] measurements (S_j S_i^-1 when made)
    kind: np.ndarray     # [m] uint8: 0 tree, 1 covisibility, 2 loop

    @property
    def n_v(self):
        return len(self.S_init)

    @property
    def n_e(self):
        return len(self.edges)


def _from13(a):
    return (float(a[12]), a[:9].reshape(3, 3).copy(), a[9:12].copy())


def make_pose_graph(name: str = "G1", seed: int = 0, mode: str = "drift", noise: float = 1e-3,
                    drift: float = 2e-3) -> PoseGraph:
    n, cov, n_loop, radius = GRAPHS[name]
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    # ground truth: camera centres on a circle, looking along the tangent
    truth = []
    for i in range(n):
        phi = 2.0 * math.pi * i / n
        c = np.array([radius * math.cos(phi), radius * math.sin(phi), 0.3 * math.sin(3 * phi)])
        yaw = phi + math.pi / 2 + 0.05 * rng.standard_normal()
        # camera z axis along the tangent: R_wc columns (x, y, z)
        z = np.array([math.cos(yaw), math.sin(yaw), 0.02 * rng.standard_normal()])
        z /= np.linalg.norm(z)
        x = np.cross(z, np.array([0.0, 0.0, 1.0]))
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        R_wc = np.stack([x, y, z], axis=1)
        truth.append(_inverse((1.0, R_wc, c)))          # world->camera
    # drifted estimates: chain the true relative motions with a multiplicative drift
    est = [truth[0]]
    for i in range(1, n):
        rel = _compose(truth[i], _inverse(truth[i - 1]))
        d = (math.exp(drift * rng.standard_normal()), _rodrigues(drift * rng.standard_normal(3)),
             drift * rng.standard_normal(3))
        est.append(_compose(_compose(d, rel), est[i - 1]))
    edges, kind = [], []
    for i in range(1, n):
        p = i - 2 if (i >= 2 and rng.random() < 0.1) else i - 1
        edges.append((p, i)); kind.append(0)
    for i in range(n):
        for j in range(i + 2, min(n, i + cov + 1)):
            if rng.random() < 0.7:
                edges.append((i, j)); kind.append(1)
    for k in range(n_loop):
        i = n - 1 - (k % max(1, n_loop // 2)) - (k // max(1, n_loop // 2)) * 2
        j = k % max(1, n_loop // 2)
        if i > j:
            edges.append((i, j)); kind.append(2)
    Ms = []
    for (i, j), kd in zip(edges, kind):
        src = truth if (mode == "exact" or kd == 2) else est
        m = _compose(src[j], _inverse(src[i]))
        if mode != "exact" and noise > 0.0:
            m = _compose((math.exp(noise * rng.standard_normal()), _rodrigues(noise * rng.standard_normal(3)),
                          noise * rng.standard_normal(3)), m)
        Ms.append(_to13(m))
    fixed = np.zeros(n, np.uint8)
    fixed[0] = 1
    return PoseGraph(name, np.stack([_to13(a) for a in est]), np.stack([_to13(a) for a in truth]), fixed,
                     np.asarray(edges, np.int32).reshape(-1, 2), np.stack(Ms), np.asarray(kind, np.uint8))
