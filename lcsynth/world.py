"""Seeded synthetic loop-closing worlds (SURVEY.md §8(d) "Synthetic worlds").

A world is a keyframe/map-point map in exactly the SoA layout of `lc_map_view`
(include/lc.h) plus one loop event (the inputs of lc_correct_sim3 / lc_fuse)
and, for the batched config, a set of projection-search hypotheses (the inputs
of lc_search_by_projection).

Structure:
  * A path (circle arc or closed circle) traversed twice. Pass A has exact
    poses; pass B has poses drifted by a Sim3 D(tau) that grows linearly along
    the pass (scale, yaw, translation), built so that pass-B map points stay
    consistent with pass-B keyframes (p_c^est = s * p_c^true).
  * Landmarks on a wall beside the path; cameras look sideways at the wall.
    5% twin landmarks (nearby, correlated descriptor) and 2% copied descriptors
    create Hamming ties and two-MPs-one-feature conflicts.
  * Observations: truth projection + N(0, 0.5^2) px, octave consistent with the
    distance (floor of the scale-space level), angle = landmark angle + N(0, 3deg).
    10% extra detections at an adjacent level with an identical descriptor
    (candidate ties broken by feature index). Clutter fills each KF to F.
  * Descriptors: landmark base (random 256 bits); observation = base xor
    Bernoulli(1/16); map point = base xor Bernoulli(1/64).
  * Map points: one per landmark per pass with >= 2 observations, ref = first
    observer, 95% of non-ref observations associated (5% left empty to exercise
    ADD), 1% flagged bad, dmax = d_ref * 1.2^oct_ref, normal = mean viewing dir.

Everything is numpy, seeded with PCG64. No oracle/CUDA arithmetic lives here;
the small Sim3 helpers below only *construct* inputs.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

N_LEVELS = 8
SCALE_FACTOR = 1.2
GRID_COLS = 64
GRID_ROWS = 48


@dataclasses.dataclass(frozen=True)
class Camera:
    model: int  # 0 pinhole, 1 Kannala-Brandt-8
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    k: tuple = (0.0, 0.0, 0.0, 0.0)

    def as_dict(self):
        return dict(model=self.model, min_x=0.0, max_x=float(self.width), min_y=0.0,
                    max_y=float(self.height), fx=self.fx, fy=self.fy, cx=self.cx,
                    cy=self.cy, k=tuple(self.k))


CAMERAS = {
    # EuRoC cam0 (EXT values, SURVEY.md §8(d) "Cameras")
    "euroc": Camera(0, 752, 480, 458.654, 457.296, 367.215, 248.375),
    # TUM-VI cam0, Kannala-Brandt 8
    "tumvi": Camera(1, 512, 512, 190.978, 190.973, 254.932, 256.897,
                    (0.0034824, 0.00071503, -0.0020532, 0.00020294)),
}


@dataclasses.dataclass(frozen=True)
class WorldConfig:
    name: str
    kf_per_pass: int
    landmarks: int
    n_feat: int
    camera: str
    wall_dist: float
    n_window: int            # 0: every pass-B KF is in the window, per-KF loop lists
    closed: bool             # closed loop path (else an arc)
    loop_covis: int = 10
    n_hyp: int = 0           # batched search hypotheses (C4)
    drift_scale: float = 0.01
    drift_yaw_deg: float = 1.0
    drift_t: tuple = (0.10, -0.05, 0.03)
    overlap: float = 2.0     # visible landmarks per KF / observed landmarks per KF


CONFIGS = {
    # BASELINE.json configs[0..4]
    "C1": WorldConfig("C1", 11, 1000, 500, "euroc", 4.0, 11, False, overlap=4.0),
    "C2": WorldConfig("C2", 150, 15000, 1000, "euroc", 4.0, 30, True, overlap=2.5),
    "C3": WorldConfig("C3", 500, 50000, 1500, "tumvi", 2.5, 40, True, overlap=2.5),
    "C4": WorldConfig("C4", 150, 15000, 1000, "euroc", 4.0, 30, True, n_hyp=32, overlap=2.5),
    "C5": WorldConfig("C5", 2500, 500000, 2000, "euroc", 4.0, 0, True, overlap=1.5),
    # small variants used by tests (ragged tails, per-KF lists, fisheye)
    "T1": WorldConfig("T1", 12, 1500, 300, "euroc", 4.0, 8, False, overlap=3.0),
    "T2": WorldConfig("T2", 16, 2500, 400, "tumvi", 2.5, 10, False, overlap=3.0),
    "T5": WorldConfig("T5", 24, 6000, 500, "euroc", 4.0, 0, True, overlap=2.0),
    # >= 296-keyframe windows (the sole-mode launch, one CTA per window keyframe) at sizes
    # the oracle finishes in seconds: pinhole and Kannala-Brandt, per-keyframe lists
    "S3": WorldConfig("S3", 320, 24000, 400, "euroc", 4.0, 0, True, overlap=1.5),
    "S3K": WorldConfig("S3K", 300, 24000, 400, "tumvi", 2.5, 0, True, overlap=1.5),
    # dense keyframes: the 4096- and 8192-feature kernel instantiations
    "T3K": WorldConfig("T3K", 8, 6000, 3000, "euroc", 4.0, 6, False, overlap=2.5),
    "T6K": WorldConfig("T6K", 6, 8000, 6000, "tumvi", 2.5, 0, True, overlap=2.5),
}

# parameter sets (th, max_hamming, ratio_num, ratio_den, check_orientation)
# EXT ORB-SLAM3 constants, SURVEY.md §8(c) A10/A11/A14.
FUSE_PARAMS = (4, 50, 0, 0, 0)
FUSE_PARAMS_CHECKS = (4, 50, 4, 5, 1)
SBP_PARAMS = [(8, 75, 0, 0, 0),   # PS2a
              (5, 50, 0, 0, 0),   # PS2b
              (3, 75, 9, 10, 1)]  # PS1 / PS3 with checks on


# ----------------------------------------------------------------------------
# small rigid-body helpers used only to construct inputs
# ----------------------------------------------------------------------------
def _rodrigues(w):
    th = float(np.linalg.norm(w))
    if th < 1e-15:
        return np.eye(3)
    k = np.asarray(w, dtype=np.float64) / th
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * (K @ K)


def _rot_z(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _compose(a, b):
    sa, Ra, ta = a
    sb, Rb, tb = b
    return (sa * sb, Ra @ Rb, sa * (Ra @ tb) + ta)


def _inverse(a):
    s, R, t = a
    return (1.0 / s, R.T, -(R.T @ t) / s)


def _to13(a):
    s, R, t = a
    out = np.empty(13, np.float64)
    out[:9] = R.reshape(-1)
    out[9:12] = t
    out[12] = s
    return out


def _noise(rng, sigma):
    """Small Sim3 perturbation, composed on the camera side (rotation about the camera)."""
    return (1.0 + sigma * rng.standard_normal(), _rodrigues(sigma * rng.standard_normal(3)),
            sigma * rng.standard_normal(3))


def _project_np(cam: Camera, pc):
    """Input-synthesis projection (numpy); returns u, v (nan where undefined)."""
    x, y, z = pc[:, 0], pc[:, 1], pc[:, 2]
    if cam.model == 0:
        with np.errstate(divide="ignore", invalid="ignore"):
            return cam.fx * x / z + cam.cx, cam.fy * y / z + cam.cy
    rho = np.sqrt(x * x + y * y)
    th = np.arctan2(rho, z)
    t2 = th * th
    k1, k2, k3, k4 = cam.k
    r = th * (1 + t2 * (k1 + t2 * (k2 + t2 * (k3 + t2 * k4))))
    with np.errstate(divide="ignore", invalid="ignore"):
        ux = np.where(rho > 0, x / rho, 0.0)
        uy = np.where(rho > 0, y / rho, 0.0)
    return cam.fx * r * ux + cam.cx, cam.fy * r * uy + cam.cy


def _rand_bits_mask(rng, n, n_and):
    """Bernoulli(2^-n_and) bit masks, shape (n, 32) uint8."""
    m = rng.integers(0, 256, size=(n, 32), dtype=np.uint8)
    for _ in range(n_and - 1):
        m &= rng.integers(0, 256, size=(n, 32), dtype=np.uint8)
    return m


@dataclasses.dataclass
class World:
    cfg: WorldConfig
    seed: int
    cam: Camera
    # --- map (lc_map_view SoA) ---
    kf_pose: np.ndarray          # (n_kf, 13) f64: R row-major, t, s (p_c = s R p + t)
    kf_cam: np.ndarray           # (n_kf,) i32
    kf_feat_begin: np.ndarray    # (n_kf+1,) i32
    feat_uv: np.ndarray          # (n_feat, 2) f32
    feat_octave: np.ndarray      # (n_feat,) u8
    feat_angle: np.ndarray       # (n_feat,) f32 degrees
    feat_desc: np.ndarray        # (n_feat, 32) u8
    feat_mp: np.ndarray          # (n_feat,) i32, -1 = empty
    mp_pos: np.ndarray           # (n_mp, 3) f32
    mp_normal: np.ndarray        # (n_mp, 3) f32
    mp_max_dist: np.ndarray      # (n_mp,) f32
    mp_desc: np.ndarray          # (n_mp, 32) u8
    mp_angle: np.ndarray         # (n_mp,) f32
    mp_ref_kf: np.ndarray        # (n_mp,) i32
    mp_flags: np.ndarray         # (n_mp,) u8 bit0 = bad
    # --- ground truth (tests only) ---
    kf_pass: np.ndarray
    feat_lm: np.ndarray
    mp_lm: np.ndarray
    mp_pass: np.ndarray
    # --- loop event ---
    cur_kf: int = 0
    window: Optional[np.ndarray] = None          # (n_w,) i32, current first
    S_cw_corr: Optional[np.ndarray] = None       # (13,)
    win_S: Optional[np.ndarray] = None           # (n_w, 13) or None (use WINDOW result)
    win_list_begin: Optional[np.ndarray] = None  # (n_w+1,) or None (shared list)
    mp_list: Optional[np.ndarray] = None         # i32, ascending unique per list
    S_opt: Optional[np.ndarray] = None           # (n_kf, 13)
    # --- batched search (C4) ---
    pair_kf: Optional[np.ndarray] = None
    pair_S: Optional[np.ndarray] = None
    pair_param: Optional[np.ndarray] = None
    pair_list_begin: Optional[np.ndarray] = None
    pair_mp_list: Optional[np.ndarray] = None
    pair_taken: Optional[np.ndarray] = None      # (sum F(pair_kf),) i32, -1 free
    list_src_begin: Optional[np.ndarray] = None  # loop lists = MPs of these keyframes (CSR)
    list_src_kf: Optional[np.ndarray] = None
    hyp_cur: Optional[np.ndarray] = None         # C4: per hypothesis, its current keyframe
    hyp_S_cw: Optional[np.ndarray] = None        # (H, 13) its loop Sim3
    hyp_win_begin: Optional[np.ndarray] = None   # (H+1,) CSR into hyp_window
    hyp_window: Optional[np.ndarray] = None      # its window (current first) = its pairs' keyframes

    @property
    def n_kf(self):
        return int(self.kf_pose.shape[0])

    @property
    def n_feat(self):
        return int(self.feat_uv.shape[0])

    @property
    def n_mp(self):
        return int(self.mp_pos.shape[0])

    def map_arrays(self):
        return dict(kf_pose=self.kf_pose, kf_cam=self.kf_cam, kf_feat_begin=self.kf_feat_begin,
                    feat_uv=self.feat_uv, feat_octave=self.feat_octave, feat_angle=self.feat_angle,
                    feat_desc=self.feat_desc, feat_mp=self.feat_mp, mp_pos=self.mp_pos,
                    mp_normal=self.mp_normal, mp_max_dist=self.mp_max_dist, mp_desc=self.mp_desc,
                    mp_angle=self.mp_angle, mp_ref_kf=self.mp_ref_kf, mp_flags=self.mp_flags)

    def n_queries(self):
        if self.win_list_begin is None:
            return int(len(self.window) * len(self.mp_list))
        return int(self.win_list_begin[-1])


def _camera_pose(c, phi, yaw_j, pitch_j):
    """Side-looking camera at centre c looking radially outward (world z up)."""
    er = np.array([math.cos(phi), math.sin(phi), 0.0])
    z = _rot_z(yaw_j) @ er
    up = np.array([0.0, 0.0, 1.0])
    z = math.cos(pitch_j) * z + math.sin(pitch_j) * up
    z /= np.linalg.norm(z)
    y = -up - np.dot(-up, z) * z
    y /= np.linalg.norm(y)
    x = np.cross(y, z)
    R_wc = np.stack([x, y, z], axis=1)
    R_cw = R_wc.T
    return (1.0, R_cw, -(R_cw @ c))


def make_world(name: str, seed: int = 0) -> World:
    cfg = CONFIGS[name]
    cam = CAMERAS[cfg.camera]
    rng = np.random.Generator(np.random.PCG64(seed * 1000003 + sum(map(ord, name))))
    K = cfg.kf_per_pass
    F = cfg.n_feat
    D = cfg.wall_dist
    n_obs_target = int(round(0.6 * F))

    # ---- geometry: visible wall strip, path length ----------------------------
    if cam.model == 0:
        w_strip = 2.0 * D * (cam.cx / cam.fx)
        band = 2.0 * D * (cam.cy / cam.fy) * 1.1
    else:
        w_strip = 2.0 * D * 2.2
        band = 2.0 * D * 1.6
    dens_target = cfg.overlap * 0.6 * F / (w_strip * band)            # landmarks per m^2 visible
    wall_len = cfg.landmarks / (dens_target * band)
    Rp = max(wall_len / (2 * math.pi), 20.0)
    Rw = Rp + D
    path_len = wall_len * Rp / Rw
    if cfg.closed:
        Rp = path_len / (2 * math.pi)
        Rw = Rp + D
        arc = 2 * math.pi
    else:
        arc = path_len / Rp
    ds = path_len / K

    # ---- landmarks --------------------------------------------------------------
    NL0 = cfg.landmarks
    n_twin = int(0.05 * NL0)
    NL = NL0 + n_twin
    lm_phi = rng.uniform(-0.5 * ds / Rp, arc + 0.5 * ds / Rp, NL0) if not cfg.closed \
        else rng.uniform(0, arc, NL0)
    lm_r = Rw + 0.03 * rng.standard_normal(NL0)
    lm_z = rng.uniform(-band / 2, band / 2, NL0)
    base = rng.integers(0, 256, size=(NL, 32), dtype=np.uint8)
    lm_ang = rng.uniform(0, 360, NL)
    # octave "size": level u with P(u) ~ 1.2^-u on [0, 8)
    uu = rng.uniform(0, 1, NL)
    a = math.log(SCALE_FACTOR)
    lm_lvl = -np.log(1 - uu * (1 - math.exp(-a * N_LEVELS))) / a
    # twins: nearby landmark with correlated descriptor (conflict generator)
    tw_src = rng.choice(NL0, n_twin, replace=False)
    lm_phi = np.concatenate([lm_phi, lm_phi[tw_src] + 0.02 * rng.standard_normal(n_twin) / Rw])
    lm_r = np.concatenate([lm_r, lm_r[tw_src] + 0.01 * rng.standard_normal(n_twin)])
    lm_z = np.concatenate([lm_z, lm_z[tw_src] + 0.02 * rng.standard_normal(n_twin)])
    base[NL0:] = base[tw_src] ^ _rand_bits_mask(rng, n_twin, 4)
    lm_ang[NL0:] = lm_ang[tw_src]
    lm_lvl[NL0:] = lm_lvl[tw_src]
    # copied descriptors (exact Hamming ties between different points)
    n_copy = int(0.02 * NL)
    cp_dst = rng.choice(NL, n_copy, replace=False)
    order_phi = np.argsort(lm_phi, kind="stable")
    rank = np.empty(NL, np.int64)
    rank[order_phi] = np.arange(NL)
    cp_src = order_phi[np.clip(rank[cp_dst] + rng.integers(1, 40, n_copy), 0, NL - 1)]
    base[cp_dst] = base[cp_src]
    lm_pos = np.stack([lm_r * np.cos(lm_phi), lm_r * np.sin(lm_phi), lm_z], axis=1)
    lm_nrm = -np.stack([np.cos(lm_phi), np.sin(lm_phi), np.zeros(NL)], axis=1)
    phi_sorted = lm_phi[order_phi]

    # ---- keyframes (true poses) --------------------------------------------------
    n_kf = 2 * K
    kf_phi = np.empty(n_kf)
    kf_true = []
    kf_c_true = np.empty((n_kf, 3))
    for p in range(2):
        for j in range(K):
            k = p * K + j
            s_path = (j + 0.5) * ds + (0.0 if p == 0 else 0.1 * ds * rng.standard_normal())
            phi = s_path / Rp
            c = np.array([Rp * math.cos(phi), Rp * math.sin(phi), 0.0])
            c = c + np.array([math.cos(phi), math.sin(phi), 0.0]) * 0.05 * rng.standard_normal()
            c[2] += 0.05 * rng.standard_normal()
            T = _camera_pose(c, phi, math.radians(3.0) * rng.standard_normal(),
                             math.radians(2.0) * rng.standard_normal())
            kf_true.append(T)
            kf_c_true[k] = c
            kf_phi[k] = phi
    kf_pass = np.repeat(np.arange(2, dtype=np.int8), K)

    # ---- drift of pass B -----------------------------------------------------------
    c0 = kf_c_true[K].copy()

    def drift(tau):
        s = 1.0 + cfg.drift_scale * tau
        R = _rot_z(math.radians(cfg.drift_yaw_deg) * tau)
        t = c0 - s * (R @ c0) + tau * np.asarray(cfg.drift_t)
        return (s, R, t)

    kf_tau = np.zeros(n_kf)
    kf_tau[K:] = np.arange(K) / max(K - 1, 1)
    kf_D = [(1.0, np.eye(3), np.zeros(3))] * K + [drift(kf_tau[K + j]) for j in range(K)]
    kf_est = []
    kf_c_est = np.empty((n_kf, 3))
    for k in range(n_kf):
        s_, R_cw, t_cw = kf_true[k]
        Dk = kf_D[k]
        c_est = Dk[0] * (Dk[1] @ kf_c_true[k]) + Dk[2]
        R_est = R_cw @ Dk[1].T
        kf_est.append((1.0, R_est, -(R_est @ c_est)))
        kf_c_est[k] = c_est

    # ---- visibility + observations -------------------------------------------------
    lateral = D * (cam.cx / cam.fx) if cam.model == 0 else D * 3.0
    dphi = (min(lateral, 20.0) + 1.5) / Rw
    obs_kf, obs_lm, obs_u, obs_v, obs_d = [], [], [], [], []
    for k in range(n_kf):
        phi = kf_phi[k]
        lo = np.searchsorted(phi_sorted, phi - dphi)
        hi = np.searchsorted(phi_sorted, phi + dphi)
        idx = order_phi[lo:hi]
        if cfg.closed:
            if phi - dphi < 0:
                idx = np.concatenate([idx, order_phi[np.searchsorted(phi_sorted, phi - dphi + 2 * math.pi):]])
            if phi + dphi > 2 * math.pi:
                idx = np.concatenate([idx, order_phi[:np.searchsorted(phi_sorted, phi + dphi - 2 * math.pi)]])
        _, R_cw, t_cw = kf_true[k]
        P = lm_pos[idx]
        pc = P @ R_cw.T + t_cw
        ok = pc[:, 2] > 0.1
        u, v = _project_np(cam, pc)
        ok &= (u >= 0) & (u < cam.width) & (v >= 0) & (v < cam.height)
        dv = kf_c_true[k] - P
        d = np.linalg.norm(dv, axis=1)
        ok &= (d >= 0.5) & (d <= 20.0)
        ok &= np.einsum("ij,ij->i", dv, lm_nrm[idx]) > 0.34 * d
        sel = np.nonzero(ok)[0]
        if len(sel) > n_obs_target:
            sel = np.sort(rng.choice(sel, n_obs_target, replace=False))
        obs_kf.append(np.full(len(sel), k, np.int64))
        obs_lm.append(idx[sel])
        obs_u.append(u[sel] + 0.5 * rng.standard_normal(len(sel)))
        obs_v.append(v[sel] + 0.5 * rng.standard_normal(len(sel)))
        obs_d.append(d[sel])
    obs_kf = np.concatenate(obs_kf)
    obs_lm = np.concatenate(obs_lm)
    obs_u = np.concatenate(obs_u)
    obs_v = np.concatenate(obs_v)
    obs_d = np.concatenate(obs_d)
    inimg = (obs_u >= 0) & (obs_u < cam.width) & (obs_v >= 0) & (obs_v < cam.height)
    obs_kf, obs_lm, obs_u, obs_v, obs_d = (x[inimg] for x in (obs_kf, obs_lm, obs_u, obs_v, obs_d))
    n_obs = len(obs_kf)
    g = lm_lvl[obs_lm] + np.log(D / obs_d) / a + 0.1 * rng.standard_normal(n_obs)
    obs_oct = np.clip(np.floor(g), 0, N_LEVELS - 1).astype(np.int64)
    obs_pass = kf_pass[obs_kf].astype(np.int64)

    # ---- map points: one per (landmark, pass) with >= 2 observations -----------------
    key = obs_pass * NL + obs_lm
    order = np.lexsort((obs_kf, key))          # by (pass, landmark), then KF
    key_s = key[order]
    starts = np.r_[0, np.nonzero(np.diff(key_s))[0] + 1]
    counts = np.diff(np.r_[starts, len(key_s)])
    good = counts >= 2
    g_starts = starts[good]
    g_counts = counts[good]
    n_mp = int(good.sum())
    mp_pass = (key_s[g_starts] // NL).astype(np.int8)
    mp_lm = (key_s[g_starts] % NL).astype(np.int32)
    # stable MP numbering: pass A first (keys sorted by pass already)
    obs_mp = np.full(n_obs, -1, np.int64)
    seg_id = np.repeat(np.arange(len(starts)), counts)
    mp_of_seg = np.full(len(starts), -1, np.int64)
    mp_of_seg[good] = np.arange(n_mp)
    obs_mp[order] = mp_of_seg[seg_id]
    ref_obs = order[g_starts]                   # first observer (lowest KF index)
    assoc = obs_mp >= 0
    drop = assoc & (rng.uniform(0, 1, n_obs) < 0.05)
    drop[ref_obs] = False
    assoc &= ~drop

    mp_ref_kf = obs_kf[ref_obs].astype(np.int32)
    # number map points in creation order (by reference keyframe), as a SLAM system
    # that triangulates points when keyframes are inserted does
    order = np.lexsort((mp_lm, mp_ref_kf))
    inv = np.empty(n_mp, np.int64)
    inv[order] = np.arange(n_mp)
    mp_pass, mp_lm, ref_obs, mp_ref_kf = mp_pass[order], mp_lm[order], ref_obs[order], mp_ref_kf[order]
    obs_mp = np.where(obs_mp >= 0, inv[np.maximum(obs_mp, 0)], -1)
    p_true = lm_pos[mp_lm]
    mp_pos = np.empty((n_mp, 3))
    for i_pass in range(2):
        m = mp_pass == i_pass
        if i_pass == 0:
            mp_pos[m] = p_true[m]
        else:
            taus = kf_tau[mp_ref_kf[m]]
            s = 1.0 + cfg.drift_scale * taus
            ang = np.radians(cfg.drift_yaw_deg) * taus
            q = p_true[m] - c0
            qr = np.stack([np.cos(ang) * q[:, 0] - np.sin(ang) * q[:, 1],
                           np.sin(ang) * q[:, 0] + np.cos(ang) * q[:, 1], q[:, 2]], axis=1)
            mp_pos[m] = s[:, None] * qr + c0 + taus[:, None] * np.asarray(cfg.drift_t)
    mp_pos += 0.01 * rng.standard_normal((n_mp, 3))
    # normal: mean viewing direction over associated observers
    a_idx = np.nonzero(assoc)[0]
    vdir = mp_pos[obs_mp[a_idx]] - kf_c_est[obs_kf[a_idx]]
    vdir /= np.linalg.norm(vdir, axis=1, keepdims=True)
    nsum = np.zeros((n_mp, 3))
    np.add.at(nsum, obs_mp[a_idx], vdir)
    mp_normal = nsum / np.linalg.norm(nsum, axis=1, keepdims=True)
    d_ref = np.linalg.norm(mp_pos - kf_c_est[mp_ref_kf], axis=1)
    mp_max_dist = d_ref * SCALE_FACTOR ** obs_oct[ref_obs]
    mp_desc = base[mp_lm] ^ _rand_bits_mask(rng, n_mp, 6)
    mp_flags = (rng.uniform(0, 1, n_mp) < 0.01).astype(np.uint8)

    # ---- features per KF: observations + extra detections + clutter ----------------
    obs_desc = base[obs_lm] ^ _rand_bits_mask(rng, n_obs, 4)
    obs_ang = np.mod(lm_ang[obs_lm] + 3.0 * rng.standard_normal(n_obs), 360.0)
    clutter_p = SCALE_FACTOR ** -np.arange(N_LEVELS, dtype=np.float64)
    clutter_p /= clutter_p.sum()
    ex = np.nonzero(rng.uniform(0, 1, n_obs) < 0.10)[0]
    n_e = len(ex)
    kf_cnt = np.bincount(obs_kf, minlength=n_kf) + np.bincount(obs_kf[ex], minlength=n_kf)
    assert kf_cnt.max() <= F
    c_cnt = F - kf_cnt
    n_c = int(c_cnt.sum())
    c_kf = np.repeat(np.arange(n_kf), c_cnt)
    all_kf = np.concatenate([obs_kf, obs_kf[ex], c_kf])
    u_all = np.concatenate([obs_u, obs_u[ex] + 0.3 * rng.standard_normal(n_e),
                            rng.uniform(0, cam.width, n_c)])
    v_all = np.concatenate([obs_v, obs_v[ex] + 0.3 * rng.standard_normal(n_e),
                            rng.uniform(0, cam.height, n_c)])
    uv_all = np.stack([np.clip(u_all, 0.0, cam.width - 1e-3),
                       np.clip(v_all, 0.0, cam.height - 1e-3)], axis=1)
    oct_all = np.concatenate([obs_oct, np.clip(obs_oct[ex] + rng.choice([-1, 1], n_e), 0, N_LEVELS - 1),
                              rng.choice(N_LEVELS, n_c, p=clutter_p)])
    ang_all = np.concatenate([obs_ang, np.mod(obs_ang[ex] + rng.standard_normal(n_e), 360.0),
                              rng.uniform(0, 360, n_c)])
    desc_all = np.concatenate([obs_desc, obs_desc[ex],
                               rng.integers(0, 256, size=(n_c, 32), dtype=np.uint8)])
    mp_all = np.concatenate([np.where(assoc, obs_mp, -1), np.full(n_e + n_c, -1)])
    lm_all = np.concatenate([obs_lm, obs_lm[ex], np.full(n_c, -1)])
    fo = np.argsort(all_kf.astype(np.int64) * (1 << 32)
                    + rng.integers(0, 1 << 32, len(all_kf), dtype=np.int64))  # random order per KF
    f_begin = np.r_[0, np.cumsum(np.full(n_kf, F))]

    w = World(
        cfg=cfg, seed=seed, cam=cam,
        kf_pose=np.stack([_to13(T) for T in kf_est]),
        kf_cam=np.zeros(n_kf, np.int32),
        kf_feat_begin=np.asarray(f_begin, np.int32),
        feat_uv=uv_all[fo].astype(np.float32),
        feat_octave=oct_all[fo].astype(np.uint8),
        feat_angle=ang_all[fo].astype(np.float32),
        feat_desc=np.ascontiguousarray(desc_all[fo]),
        feat_mp=mp_all[fo].astype(np.int32),
        mp_pos=mp_pos.astype(np.float32),
        mp_normal=mp_normal.astype(np.float32),
        mp_max_dist=mp_max_dist.astype(np.float32),
        mp_desc=np.ascontiguousarray(mp_desc),
        mp_angle=obs_ang[ref_obs].astype(np.float32),
        mp_ref_kf=mp_ref_kf,
        mp_flags=mp_flags,
        kf_pass=kf_pass,
        feat_lm=lm_all[fo].astype(np.int32),
        mp_lm=mp_lm,
        mp_pass=mp_pass,
    )

    # ---- loop event --------------------------------------------------------------
    ideal = [None] * n_kf
    for k in range(n_kf):
        ideal[k] = _compose(kf_est[k], kf_D[k]) if k >= K else kf_est[k]
    cur = n_kf - 1
    w.cur_kf = cur
    w.S_cw_corr = _to13(_compose(_noise(rng, 1e-3), ideal[cur]))
    w.S_opt = np.stack([_to13(_compose(_noise(rng, 1e-4), ideal[k])) if k >= K else _to13(kf_est[k])
                        for k in range(n_kf)])
    covis = _covisibility(w) if (cfg.n_window > 0 or cfg.n_hyp > 0) else None
    if cfg.n_window > 0:
        w.window = np.asarray([cur] + _top_covisible(covis, cur, cfg.n_window - 1, lambda j: j >= K),
                              np.int32)
        matched = cur - K
        loop_kfs = [matched] + _top_covisible(covis, matched, cfg.loop_covis, lambda j: j < K)
        w.mp_list = _kf_mps(w, loop_kfs)
        w.list_src_begin = np.asarray([0, len(loop_kfs)], np.int32)   # one shared list
        w.list_src_kf = np.asarray(loop_kfs, np.int32)
    else:
        w.window = np.asarray([cur] + list(range(K, n_kf - 1)), np.int32)
        lists, begin, src, sbeg = [], [0], [], [0]
        for k in w.window:
            j = int(k) - K
            nb = [(j + o) % K if cfg.closed else min(max(j + o, 0), K - 1) for o in range(-5, 6)]
            lst = _kf_mps(w, sorted(set(nb)))
            lists.append(lst)
            begin.append(begin[-1] + len(lst))
            src += sorted(set(nb))
            sbeg.append(len(src))
        w.list_src_begin = np.asarray(sbeg, np.int32)   # the lists' source keyframes (CSR)
        w.list_src_kf = np.asarray(src, np.int32)
        w.win_list_begin = np.asarray(begin, np.int32)
        w.mp_list = np.concatenate(lists).astype(np.int32)
        w.win_S = np.stack([_to13(_compose(_noise(rng, 1e-3), ideal[int(k)])) for k in w.window])

    if cfg.n_hyp > 0:
        _make_hypotheses(w, rng, covis, kf_est, ideal, K)
    return w


def _covisibility(w: World):
    import scipy.sparse as sp
    kf_of_feat = np.repeat(np.arange(w.n_kf), np.diff(w.kf_feat_begin))
    m = w.feat_mp >= 0
    A = sp.csr_matrix((np.ones(int(m.sum()), np.int32), (kf_of_feat[m], w.feat_mp[m])),
                      shape=(w.n_kf, w.n_mp))
    A.data[:] = 1
    C = (A @ A.T).toarray()
    np.fill_diagonal(C, 0)
    return C


def _top_covisible(C, k, n, allow):
    cand = [j for j in range(C.shape[0]) if j != k and allow(j) and C[k, j] > 0]
    cand.sort(key=lambda j: (-C[k, j], j))
    return cand[:n]


def _kf_mps(w: World, kfs):
    parts = [w.feat_mp[w.kf_feat_begin[k]:w.kf_feat_begin[k + 1]] for k in kfs]
    allm = np.concatenate(parts) if parts else np.zeros(0, np.int32)
    return np.unique(allm[allm >= 0]).astype(np.int32)


def _make_hypotheses(w: World, rng, covis, kf_est, ideal, K):
    H = w.cfg.n_hyp
    pair_kf, pair_S, pair_param, lists, begin = [], [], [], [], [0]
    hyp_cur, hyp_S, pair_hyp = [], [], []
    for h in range(H):
        j = int(round((h + 0.5) * K / H)) % K
        cur = K + j
        S_cw = _compose(_noise(rng, 1e-3), ideal[cur])
        hyp_cur.append(cur)
        hyp_S.append(_to13(S_cw))
        loop_kfs = [j] + _top_covisible(covis, j, w.cfg.loop_covis, lambda x: x < K)
        lst = _kf_mps(w, loop_kfs)
        for kk in [cur] + _top_covisible(covis, cur, 3, lambda x: x >= K):
            S_ic = _compose(kf_est[kk], _inverse(kf_est[cur]))
            pair_kf.append(kk)
            pair_hyp.append(h)
            pair_S.append(_to13(_compose(S_ic, S_cw)))
            pair_param.append(h % 3)
            lists.append(lst)
            begin.append(begin[-1] + len(lst))
    w.pair_kf = np.asarray(pair_kf, np.int32)
    w.pair_S = np.stack(pair_S)
    # the hypotheses' own window corrections (SURVEY §8(d) C4 "32 lc_correct_sim3 dry runs"):
    # hypothesis h = (current KF, S_cw, window = its 4 pairs' keyframes, current first)
    w.hyp_cur = np.asarray(hyp_cur, np.int32)
    w.hyp_S_cw = np.stack(hyp_S)
    w.hyp_window = w.pair_kf.copy()
    w.hyp_win_begin = np.searchsorted(np.asarray(pair_hyp), np.arange(H + 1)).astype(np.int32)
    w.pair_param = np.asarray(pair_param, np.int32)
    w.pair_list_begin = np.asarray(begin, np.int32)
    w.pair_mp_list = np.concatenate(lists).astype(np.int32)
    taken = []
    for p, kk in enumerate(w.pair_kf):
        nf = int(w.kf_feat_begin[kk + 1] - w.kf_feat_begin[kk])
        t = np.full(nf, -1, np.int32)
        if w.pair_param[p] == 1:
            lst = w.pair_mp_list[w.pair_list_begin[p]:w.pair_list_begin[p + 1]]
            sel = rng.uniform(0, 1, nf) < 0.05
            if len(lst):
                t[sel] = rng.choice(lst, int(sel.sum()))
        taken.append(t)
    w.pair_taken = np.concatenate(taken)
