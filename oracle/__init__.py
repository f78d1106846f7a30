"""ctypes wrapper of the CPU oracle (oracle/lc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product package
(paper_2603_17201_b200) never imports this module, and this module never
imports the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

COUNTER_NAMES = [
    "queries", "skip_bad", "skip_found", "cull_depth", "cull_bounds", "cull_dist",
    "cull_angle", "candidates", "no_cand", "over_th", "ratio_rej", "proposals",
    "winners", "orient_rej", "add", "victim_prop", "loop_skip", "bad_slot",
    "victims", "rewired", "dup_cleared", "added", "corr_kf", "corr_mp",
    "refresh_mp", "refresh_obs", "conn_kf", "conn_edges", "ransac_hyp", "ransac_inliers",
    "refine_iters", "refine_inliers", "pgo_iters", "pgo_accepted", "pgo_solver_iters", "pgo_stop",
    "pgo_band", "forced", "edge_amb", "pgo_cr_levels",   # pgo_cr_levels: a device-solver counter, always 0 here
]
NONE64 = np.iinfo(np.int64).max

# query status codes
Q_BAD, Q_FOUND, Q_DEPTH, Q_BOUNDS, Q_DIST, Q_ANGLE = -1, -2, -3, -4, -5, -6


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -ffp-contract=off so fp64 runs in written order)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


class _Camera(C.Structure):
    _fields_ = [("model", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("k", C.c_double * 4),
                ("min_x", C.c_double), ("max_x", C.c_double), ("min_y", C.c_double),
                ("max_y", C.c_double)]


class _Params(C.Structure):
    _fields_ = [("th", C.c_int32), ("max_hamming", C.c_int32), ("ratio_num", C.c_int32),
                ("ratio_den", C.c_int32), ("check_orientation", C.c_int32)]


class _Map(C.Structure):
    _fields_ = [("n_kf", C.c_int32), ("n_feat", C.c_int32), ("n_mp", C.c_int32),
                ("n_levels", C.c_int32), ("scale_factor", C.c_double),
                ("kf_pose", C.c_void_p), ("kf_cam", C.c_void_p), ("kf_feat_begin", C.c_void_p),
                ("feat_uv", C.c_void_p), ("feat_octave", C.c_void_p), ("feat_angle", C.c_void_p),
                ("feat_desc", C.c_void_p), ("feat_mp", C.c_void_p), ("mp_pos", C.c_void_p),
                ("mp_normal", C.c_void_p), ("mp_max_dist", C.c_void_p), ("mp_desc", C.c_void_p),
                ("mp_angle", C.c_void_p), ("mp_ref_kf", C.c_void_p), ("mp_flags", C.c_void_p),
                ("mp_replaced_by", C.c_void_p), ("mp_nobs", C.c_void_p),
                ("mp_corr_ref", C.c_void_p), ("kf_in_window", C.c_void_p),
                ("kf_S_corr", C.c_void_p), ("cams", C.c_void_p), ("n_cams", C.c_int32)]


class _QRes(C.Structure):
    _fields_ = [("status", C.c_int32), ("u", C.c_double), ("v", C.c_double),
                ("level", C.c_int32), ("radius", C.c_double), ("ncand", C.c_int32),
                ("best_f", C.c_int32), ("best_h", C.c_int32), ("second_h", C.c_int32),
                ("edge", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_hamming.restype = C.c_int
        _lib.orc_predict_level.restype = C.c_int
        _lib.orc_predict_level.argtypes = [C.c_double, C.c_double, C.c_void_p, C.c_int32]
        for fn in ("orc_correct_window", "orc_correct_all", "orc_fuse", "orc_search_by_projection",
                   "orc_refresh", "orc_update_connections", "orc_sim3_ransac", "orc_sim3_refine", "orc_pgo",
                   "orc_correct_window_batch", "orc_fuse_plan_grid"):
            getattr(_lib, fn).restype = C.c_int
        _lib.orc_loop_lists.restype = C.c_int64
        _lib.orc_grid_build.restype = C.c_void_p
        _lib.orc_grid_free.argtypes = [C.c_void_p]
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def make_camera(cam) -> _Camera:
    d = cam.as_dict() if hasattr(cam, "as_dict") else dict(cam)
    c = _Camera()
    c.model = d["model"]
    c.fx, c.fy, c.cx, c.cy = d["fx"], d["fy"], d["cx"], d["cy"]
    for i in range(4):
        c.k[i] = d["k"][i]
    c.min_x, c.max_x, c.min_y, c.max_y = d["min_x"], d["max_x"], d["min_y"], d["max_y"]
    return c


def make_params(p) -> _Params:
    th, mh, rn, rd, co = p
    return _Params(th, mh, rn, rd, co)


# ----------------------------------------------------------------------------
# primitives (pinned directly by tests/test_oracle_pins.py)
# ----------------------------------------------------------------------------
def hamming(a, b) -> int:
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    return int(lib().orc_hamming(_p(a), _p(b)))


def _sim3_call(fn, *args):
    out = np.zeros(13 if fn != "orc_sim3_apply" else 3, np.float64)
    arrs = [np.ascontiguousarray(a, np.float64) for a in args]
    getattr(lib(), fn)(*[_p(a) for a in arrs], _p(out))
    return out


def sim3_apply(S, p):
    return _sim3_call("orc_sim3_apply", S, p)


def sim3_compose(A, B):
    return _sim3_call("orc_sim3_compose", A, B)


def sim3_inverse(S):
    return _sim3_call("orc_sim3_inverse", S)


def sim3_se3(S):
    return _sim3_call("orc_sim3_se3", S)


def project(cam, pc):
    c = make_camera(cam)
    pc = np.ascontiguousarray(pc, np.float64)
    uv = np.zeros(2, np.float64)
    lib().orc_project(C.byref(c), _p(pc), _p(uv))
    return uv


def jacobi4(A):
    """Eigenvalues / eigenvector columns of a symmetric 4x4 (oracle's Jacobi, A42)."""
    A = np.ascontiguousarray(A, np.float64).reshape(4, 4)
    ev = np.zeros(4, np.float64)
    V = np.zeros((4, 4), np.float64)
    lib().orc_jacobi4(_p(A), _p(ev), _p(V))
    return ev, V


def horn(P1, P2, fix_scale=False):
    """Closed-form similarity S12 (p1 ~ s R p2 + t) of all correspondences (A42)."""
    P1 = np.ascontiguousarray(P1, np.float64).reshape(-1, 3)
    P2 = np.ascontiguousarray(P2, np.float64).reshape(-1, 3)
    sel = np.arange(len(P1), dtype=np.int32)
    S = np.zeros(13, np.float64)
    lib().orc_horn(C.c_int32(len(P1)), _p(sel), _p(P1), _p(P2), C.c_int32(int(fix_scale)), _p(S))
    return S


def sim3_retract(d, S):
    """S <- (Cayley(w), tau, 1 + sig) o S for d = (w, tau, sig) (A45)."""
    out = np.zeros(13, np.float64)
    lib().orc_sim3_retract(_p(np.ascontiguousarray(d, np.float64)), _p(np.ascontiguousarray(S, np.float64)),
                           _p(out))
    return out


def scale_table(L=8, f=1.2):
    out = np.zeros(L, np.float64)
    lib().orc_scale_table(C.c_int32(L), C.c_double(f), _p(out))
    return out


def predict_level(d, dmax, L=8, f=1.2):
    st = scale_table(L, f)
    return int(lib().orc_predict_level(C.c_double(d), C.c_double(dmax), _p(st), C.c_int32(L)))


# ----------------------------------------------------------------------------
# map state
# ----------------------------------------------------------------------------
class _Grid:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            lib().orc_grid_free(self.h)
            self.h = None

class OracleMap:
    """Mutable copy of a world's map plus the loop state, driven by the C oracle."""

    def __init__(self, world=None, *, arrays=None, cams=None, n_levels=8, scale_factor=1.2):
        a = arrays if arrays is not None else world.map_arrays()
        cams = cams if cams is not None else [world.cam]
        self.kf_pose = np.array(a["kf_pose"], np.float64, order="C").reshape(-1, 13)
        self.kf_cam = np.ascontiguousarray(a["kf_cam"], np.int32)
        self.kf_feat_begin = np.ascontiguousarray(a["kf_feat_begin"], np.int32)
        self.feat_uv = np.ascontiguousarray(a["feat_uv"], np.float32).reshape(-1, 2)
        self.feat_octave = np.ascontiguousarray(a["feat_octave"], np.uint8)
        self.feat_angle = np.ascontiguousarray(a["feat_angle"], np.float32)
        self.feat_desc = np.ascontiguousarray(a["feat_desc"], np.uint8).reshape(-1, 32)
        self.feat_mp = np.array(a["feat_mp"], np.int32)
        self.mp_pos = np.array(a["mp_pos"], np.float32).reshape(-1, 3)
        self.mp_normal = np.array(a["mp_normal"], np.float32).reshape(-1, 3)      # mutable copies
        self.mp_max_dist = np.array(a["mp_max_dist"], np.float32)
        self.mp_desc = np.array(a["mp_desc"], np.uint8).reshape(-1, 32)
        self.mp_angle = np.ascontiguousarray(a["mp_angle"], np.float32)
        self.mp_ref_kf = np.ascontiguousarray(a["mp_ref_kf"], np.int32)
        self.mp_flags = np.array(a["mp_flags"], np.uint8)
        n_kf, n_mp = self.kf_pose.shape[0], self.mp_pos.shape[0]
        self.mp_replaced_by = np.full(n_mp, -1, np.int32)
        self.mp_nobs = np.bincount(self.feat_mp[self.feat_mp >= 0], minlength=n_mp).astype(np.int32)
        self.mp_corr_ref = np.full(n_mp, -1, np.int32)
        self.kf_in_window = np.zeros(n_kf, np.int32)
        self.kf_S_corr = np.zeros((n_kf, 13), np.float64)
        self._cams = (_Camera * len(cams))(*[make_camera(c) for c in cams])
        m = _Map()
        m.n_kf, m.n_feat, m.n_mp = n_kf, self.feat_uv.shape[0], n_mp
        m.n_levels, m.scale_factor = n_levels, scale_factor
        for name in ("kf_pose", "kf_cam", "kf_feat_begin", "feat_uv", "feat_octave", "feat_angle",
                     "feat_desc", "feat_mp", "mp_pos", "mp_normal", "mp_max_dist", "mp_desc",
                     "mp_angle", "mp_ref_kf", "mp_flags", "mp_replaced_by", "mp_nobs",
                     "mp_corr_ref", "kf_in_window", "kf_S_corr"):
            setattr(m, name, getattr(self, name).ctypes.data)
        m.cams = C.cast(self._cams, C.c_void_p).value
        m.n_cams = len(cams)
        self._m = m

    @property
    def n_kf(self):
        return self.kf_pose.shape[0]

    @property
    def n_mp(self):
        return self.mp_pos.shape[0]

    def n_feat_of(self, k):
        return int(self.kf_feat_begin[k + 1] - self.kf_feat_begin[k])

    # -- single query (pins) --------------------------------------------------
    def query(self, k, S_kw, q, params, taken=None, mode=0):
        r = _QRes()
        S = np.ascontiguousarray(S_kw, np.float64)
        t = None if taken is None else np.ascontiguousarray(taken, np.int32)
        prm = make_params(params)
        lib().orc_query(C.byref(self._m), C.c_int32(k), _p(S), C.c_int32(q), C.byref(prm),
                        _p(t), C.c_int32(mode), C.byref(r))
        return {f: getattr(r, f) for f, _ in _QRes._fields_}

    # -- O3 ------------------------------------------------------------------
    def correct_window(self, cur_kf, S_cw_corr, window):
        window = np.ascontiguousarray(window, np.int32)
        S = np.ascontiguousarray(S_cw_corr, np.float64)
        out_S = np.zeros((len(window), 13), np.float64)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        rc = lib().orc_correct_window(C.byref(self._m), C.c_int32(cur_kf), _p(S),
                                      C.c_int32(len(window)), _p(window), _p(out_S), _p(cnt))
        if rc != 0:
            raise ValueError("orc_correct_window: invalid arguments")
        return out_S, dict(zip(COUNTER_NAMES, cnt.tolist()))

    # -- O3' -----------------------------------------------------------------
    def correct_window_batch(self, cur_kf, S_cw_corr, window_begin, window, capacity=None):
        """Dry-run window corrections of several hypotheses (no write-back): returns
        (S_corr [sum window, 13], mp_begin [n_batch + 1], mp_idx, mp_pos [n, 3], counts)."""
        cur = np.ascontiguousarray(cur_kf, np.int32)
        nb = len(cur)
        S = np.ascontiguousarray(S_cw_corr, np.float64).reshape(nb, 13)
        wb = np.ascontiguousarray(window_begin, np.int32)
        win = np.ascontiguousarray(window, np.int32)
        out_S = np.zeros((len(win), 13), np.float64)
        mb = np.zeros(nb + 1, np.int32)
        cap = nb * self.n_mp if capacity is None else int(capacity)
        idx = np.zeros(max(cap, 1), np.int32)
        pos = np.zeros((max(cap, 1), 3), np.float32)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        rc = lib().orc_correct_window_batch(C.byref(self._m), C.c_int32(nb), _p(cur), _p(S), _p(wb), _p(win),
                                            _p(out_S), _p(mb), _p(idx), _p(pos), C.c_int64(cap), _p(cnt))
        if rc == -1:
            raise ValueError("orc_correct_window_batch: invalid arguments")
        if rc == -2:
            raise OverflowError(f"capacity {cap} < {int(mb[-1])} corrected points")
        n = int(mb[-1])
        return out_S, mb, idx[:n], pos[:n], dict(zip(COUNTER_NAMES, cnt.tolist()))

    # -- O10 -----------------------------------------------------------------
    def correct_all(self, S_opt):
        S = np.ascontiguousarray(S_opt, np.float64).reshape(-1, 13)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        lib().orc_correct_all(C.byref(self._m), _p(S), _p(cnt))
        return dict(zip(COUNTER_NAMES, cnt.tolist()))

    # -- O4-O9 ---------------------------------------------------------------
    def window_feat_total(self, window):
        return int(sum(self.n_feat_of(int(k)) for k in window))

    def fuse(self, window, mp_list, params, *, window_S=None, win_list_begin=None, phase=3,
             w_lo=0, w_hi=None, winner=None, victim=None, debug=False, cur_kf=-1, forced_mp=None):
        window = np.ascontiguousarray(window, np.int32)
        n_w = len(window)
        w_hi = n_w if w_hi is None else w_hi
        mp_list = np.ascontiguousarray(mp_list, np.int32)
        wb = None if win_list_begin is None else np.ascontiguousarray(win_list_begin, np.int32)
        wS = None if window_S is None else np.ascontiguousarray(window_S, np.float64).reshape(-1, 13)
        nwf = self.window_feat_total(window)
        winner = np.full(nwf, NONE64, np.int64) if winner is None else winner
        victim = np.full(self.n_mp, NONE64, np.int64) if victim is None else victim
        action = np.zeros(nwf, np.int8)
        nq = int(wb[-1]) if wb is not None else n_w * len(mp_list)
        dbg = {}
        if debug:
            dbg = dict(status=np.zeros(nq, np.int32), best=np.zeros(nq, np.int64),
                       uv=np.zeros((nq, 2), np.float64), ncand=np.zeros(nq, np.int32),
                       edge=np.zeros(nq, np.uint8))
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        prm = make_params(params)
        if not (0 <= w_lo <= w_hi <= n_w):
            raise ValueError("bad shard range")
        fm = None if forced_mp is None else np.ascontiguousarray(forced_mp, np.int32)
        if fm is not None and len(fm) != self.n_feat_of(int(cur_kf)):
            raise ValueError("forced_mp must have F(cur_kf) entries")
        rc = lib().orc_fuse(C.byref(self._m), C.c_int32(phase), C.c_int32(w_lo), C.c_int32(w_hi),
                       C.c_int32(n_w), _p(window), _p(wS), _p(wb), _p(mp_list),
                       C.c_int32(len(mp_list)), C.byref(prm), C.c_int32(int(cur_kf)), _p(fm),
                       _p(winner), _p(victim), _p(action),
                       _p(dbg.get("status")), _p(dbg.get("best")), _p(dbg.get("uv")),
                       _p(dbg.get("ncand")), _p(dbg.get("edge")), _p(cnt))
        if rc != 0:
            raise ValueError("orc_fuse: invalid arguments")
        return dict(winner=winner, victim=victim, action=action,
                    counts=dict(zip(COUNTER_NAMES, cnt.tolist())), **dbg)

    # -- loop map-point lists ------------------------------------------------
    def loop_lists(self, src_begin, src_kf):
        """List l = ascending unique map points held by keyframes src_kf[src_begin[l]:src_begin[l+1]]:
        returns (begin [n + 1], lists)."""
        sb = np.ascontiguousarray(src_begin, np.int32)
        sk = np.ascontiguousarray(src_kf, np.int32)
        n = len(sb) - 1
        cap = int(sum(self.n_feat_of(int(k)) for k in sk))
        ob = np.zeros(n + 1, np.int32)
        ol = np.zeros(max(cap, 1), np.int32)
        tot = lib().orc_loop_lists(C.byref(self._m), C.c_int32(n), _p(sb), _p(sk), _p(ob), _p(ol), C.c_int64(cap))
        if tot < 0:
            raise ValueError("orc_loop_lists: invalid arguments")
        return ob, ol[:tot]

    # -- timing-only grid / threaded PLAN (bench.py cpu_baseline) --------------
    def grid(self, cols=64, rows=48):
        """Per-keyframe cell grid for fuse_plan_grid (built once per map, untimed)."""
        h = lib().orc_grid_build(C.byref(self._m), C.c_int32(cols), C.c_int32(rows))
        return _Grid(h)

    def fuse_plan_grid(self, grid, n_threads, window, mp_list, params, *, window_S=None, win_list_begin=None):
        window = np.ascontiguousarray(window, np.int32)
        mp_list = np.ascontiguousarray(mp_list, np.int32)
        wb = None if win_list_begin is None else np.ascontiguousarray(win_list_begin, np.int32)
        wS = None if window_S is None else np.ascontiguousarray(window_S, np.float64).reshape(-1, 13)
        winner = np.full(self.window_feat_total(window), NONE64, np.int64)
        victim = np.full(self.n_mp, NONE64, np.int64)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        prm = make_params(params)
        rc = lib().orc_fuse_plan_grid(C.byref(self._m), C.c_void_p(grid.h), C.c_int32(n_threads),
                                      C.c_int32(len(window)), _p(window), _p(wS), _p(wb), _p(mp_list),
                                      C.c_int32(len(mp_list)), C.byref(prm), _p(winner), _p(victim), _p(cnt))
        if rc != 0:
            raise ValueError("orc_fuse_plan_grid: invalid arguments")
        return dict(winner=winner, victim=victim, counts=dict(zip(COUNTER_NAMES, cnt.tolist())))

    # -- batched projection search -------------------------------------------
    def search_by_projection(self, pair_kf, pair_S, pair_param, params, pair_list_begin, mp_list,
                             pair_taken=None, debug=False):
        pair_kf = np.ascontiguousarray(pair_kf, np.int32)
        pair_S = np.ascontiguousarray(pair_S, np.float64).reshape(-1, 13)
        pair_param = np.ascontiguousarray(pair_param, np.int32)
        plb = np.ascontiguousarray(pair_list_begin, np.int32)
        mp_list = np.ascontiguousarray(mp_list, np.int32)
        taken = None if pair_taken is None else np.ascontiguousarray(pair_taken, np.int32)
        prms = (_Params * len(params))(*[make_params(p) for p in params])
        ntot = int(sum(self.n_feat_of(int(k)) for k in pair_kf))
        out_mp = np.zeros(ntot, np.int32)
        out_dist = np.zeros(ntot, np.int32)
        nq = int(plb[-1])
        dbg = {}
        if debug:
            dbg = dict(best=np.zeros(nq, np.int64), uv=np.zeros((nq, 2), np.float64),
                       ncand=np.zeros(nq, np.int32), edge=np.zeros(nq, np.uint8))
        cnt = np.zeros((len(pair_kf), len(COUNTER_NAMES)), np.int64)
        lib().orc_search_by_projection(C.byref(self._m), C.c_int32(len(pair_kf)), _p(pair_kf),
                                       _p(pair_S), _p(pair_param), prms, _p(plb), _p(mp_list),
                                       _p(taken), _p(out_mp), _p(out_dist), _p(dbg.get("best")),
                                       _p(dbg.get("uv")), _p(dbg.get("ncand")),
                                       _p(dbg.get("edge")), _p(cnt))
        return dict(feat_mp=out_mp, feat_dist=out_dist, counts=cnt, **dbg)

    # -- O11 -----------------------------------------------------------------
    def refresh(self, mp_idx=None, what=3):
        """Map-point refresh (descriptor: what & 1, normal + depth range: what & 2)."""
        idx = None if mp_idx is None else np.ascontiguousarray(mp_idx, np.int32)
        n = self.n_mp if idx is None else len(idx)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        rc = lib().orc_refresh(C.byref(self._m), C.c_int32(n), _p(idx), C.c_int32(what), _p(cnt))
        if rc != 0:
            raise ValueError("orc_refresh: invalid arguments")
        return dict(zip(COUNTER_NAMES, cnt.tolist()))

    # -- O12 -----------------------------------------------------------------
    def update_connections(self, kf_idx=None, th=15, max_edges=64):
        """Covisibility edges of the given keyframes (None: all): (n_edges, kf, weight)
        with kf / weight [n, max_edges] (rows valid up to min(n_edges, max_edges))."""
        idx = None if kf_idx is None else np.ascontiguousarray(kf_idx, np.int32)
        n = self.n_kf if idx is None else len(idx)
        out_n = np.zeros(n, np.int32)
        out_kf = np.full((n, max_edges), -1, np.int32)
        out_w = np.zeros((n, max_edges), np.int32)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        rc = lib().orc_update_connections(C.byref(self._m), C.c_int32(n), _p(idx), C.c_int32(th),
                                          C.c_int32(max_edges), _p(out_n), _p(out_kf), _p(out_w), _p(cnt))
        if rc != 0:
            raise ValueError("orc_update_connections: invalid arguments")
        return out_n, out_kf, out_w, dict(zip(COUNTER_NAMES, cnt.tolist()))

    # -- O13 -----------------------------------------------------------------
    def sim3_ransac(self, prob_begin, P1, P2, uv1, uv2, sig1, sig2, cam1, cam2, samples,
                    chi2=9.210, fix_scale=False, refit=True):
        """Batched Sim3 RANSAC: returns (S [n_prob, 13], inliers [n_prob], mask [n_corr], counts)."""
        pb = np.ascontiguousarray(prob_begin, np.int32)
        n_prob = len(pb) - 1
        P1 = np.ascontiguousarray(P1, np.float64).reshape(-1, 3)
        P2 = np.ascontiguousarray(P2, np.float64).reshape(-1, 3)
        uv1 = np.ascontiguousarray(uv1, np.float32).reshape(-1, 2)
        uv2 = np.ascontiguousarray(uv2, np.float32).reshape(-1, 2)
        sig1 = np.ascontiguousarray(sig1, np.float32)
        sig2 = np.ascontiguousarray(sig2, np.float32)
        cam1 = np.ascontiguousarray(cam1, np.int32)
        cam2 = np.ascontiguousarray(cam2, np.int32)
        smp = np.ascontiguousarray(samples, np.int32).reshape(n_prob, -1, 3)
        n_iter = smp.shape[1]
        S = np.zeros((n_prob, 13), np.float64)
        inl = np.zeros(n_prob, np.int32)
        mask = np.zeros(len(P1), np.uint8)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        lib().orc_sim3_ransac(C.byref(self._m), C.c_int32(n_prob), _p(pb), _p(P1), _p(P2), _p(uv1),
                              _p(uv2), _p(sig1), _p(sig2), _p(cam1), _p(cam2), _p(smp), C.c_int32(n_iter),
                              C.c_double(chi2), C.c_int32(int(fix_scale)), C.c_int32(int(refit)), _p(S),
                              _p(inl), _p(mask), _p(cnt))
        return S, inl, mask, dict(zip(COUNTER_NAMES, cnt.tolist()))

    # -- O14 -----------------------------------------------------------------
    def sim3_refine(self, prob_begin, P1, P2, uv1, uv2, sig1, sig2, cam1, cam2, S_init, max_iter=10,
                    th2=10.0, lam=1e-6):
        """Gauss-Newton Sim3 refinement: (S [n_prob, 13], inliers [n_prob], mask [n_corr], counts)."""
        pb = np.ascontiguousarray(prob_begin, np.int32)
        n_prob = len(pb) - 1
        P1 = np.ascontiguousarray(P1, np.float64).reshape(-1, 3)
        P2 = np.ascontiguousarray(P2, np.float64).reshape(-1, 3)
        uv1 = np.ascontiguousarray(uv1, np.float32).reshape(-1, 2)
        uv2 = np.ascontiguousarray(uv2, np.float32).reshape(-1, 2)
        sig1 = np.ascontiguousarray(sig1, np.float32)
        sig2 = np.ascontiguousarray(sig2, np.float32)
        cam1 = np.ascontiguousarray(cam1, np.int32)
        cam2 = np.ascontiguousarray(cam2, np.int32)
        S0 = np.ascontiguousarray(S_init, np.float64).reshape(n_prob, 13)
        S = np.zeros((n_prob, 13), np.float64)
        inl = np.zeros(n_prob, np.int32)
        mask = np.zeros(len(P1), np.uint8)
        cnt = np.zeros(len(COUNTER_NAMES), np.int64)
        lib().orc_sim3_refine(C.byref(self._m), C.c_int32(n_prob), _p(pb), _p(P1), _p(P2), _p(uv1), _p(uv2),
                              _p(sig1), _p(sig2), _p(cam1), _p(cam2), _p(S0), C.c_int32(max_iter),
                              C.c_double(th2), C.c_double(lam), _p(S), _p(inl), _p(mask), _p(cnt))
        return S, inl, mask, dict(zip(COUNTER_NAMES, cnt.tolist()))


# ----------------------------------------------------------------------------
# O15: essential-graph Sim3 pose-graph optimisation (readings A49-A53)
# ----------------------------------------------------------------------------
class _PgoParams(C.Structure):
    _fields_ = [("max_iter", C.c_int32), ("cg_max_iter", C.c_int32), ("lambda0", C.c_double),
                ("eps_dx", C.c_double), ("eps_chi2", C.c_double), ("cg_tol", C.c_double)]


PGO_STOP = {1: "dx", 2: "chi2", 3: "max_iter", 4: "lambda", 5: "zero"}


def pgo_exp(x):
    """Sim3 exponential of x = (omega, upsilon, sigma) (A49)."""
    out = np.zeros(13, np.float64)
    lib().orc_pgo_exp(_p(np.ascontiguousarray(x, np.float64)), _p(out))
    return out


def pgo_log(S):
    """Sim3 logarithm (A49): (omega, upsilon, sigma)."""
    out = np.zeros(7, np.float64)
    lib().orc_pgo_log(_p(np.ascontiguousarray(S, np.float64)), _p(out))
    return out


def pgo_edge(M, Si, Sj):
    """Residual e = log(M o S_i o S_j^-1) and its dual-number Jacobians (A50):
    (e [7], J_i [7, 7], J_j [7, 7]), J[r, k] = d e_r / d delta_k."""
    e = np.zeros(7, np.float64)
    Ji = np.zeros((7, 7), np.float64)
    Jj = np.zeros((7, 7), np.float64)
    lib().orc_pgo_edge(*[_p(np.ascontiguousarray(a, np.float64)) for a in (M, Si, Sj)], _p(e), _p(Ji), _p(Jj))
    return e, Ji, Jj


def pgo(S_init, fixed, edges, M, max_iter=20, lambda0=1e-4, eps_dx=1e-8, eps_chi2=1e-10):
    """Levenberg-Marquardt essential-graph optimisation with dense LDL^T (A51-A53).
    Returns (S [n_v, 13], trace [iters, 6], (chi2_0, chi2_final), counts)."""
    S0 = np.ascontiguousarray(S_init, np.float64).reshape(-1, 13)
    n_v = len(S0)
    fx = np.ascontiguousarray(fixed, np.uint8)
    E = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    Mm = np.ascontiguousarray(M, np.float64).reshape(-1, 13)
    prm = _PgoParams(int(max_iter), 0, float(lambda0), float(eps_dx), float(eps_chi2), 0.0)
    S = np.zeros((n_v, 13), np.float64)
    tr = np.zeros((max(int(max_iter), 1), 6), np.float64)
    c2 = np.zeros(2, np.float64)
    cnt = np.zeros(len(COUNTER_NAMES), np.int64)
    lib().orc_pgo(C.c_int32(n_v), _p(S0), _p(fx), C.c_int32(len(E)), _p(E), _p(Mm), C.byref(prm), _p(S),
                  _p(tr), _p(c2), _p(cnt))
    cd = dict(zip(COUNTER_NAMES, cnt.tolist()))
    return S, tr[:cd["pgo_iters"]], (float(c2[0]), float(c2[1])), cd
