"""Thin Python binding of liblc (include/lc.h): same entry points, argument
marshalling only. Arrays may be torch tensors (CPU or CUDA) or numpy arrays;
every step of the path runs in liblc's kernels. Outputs are torch CUDA tensors
(asynchronous, on the current stream) unless `host=True` (numpy, synchronised).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import (COUNTER_NAMES, LC_CORRECT_ALL, LC_CORRECT_WINDOW, LC_FUSE_ALL, LC_FUSE_APPLY,
                   LC_FUSE_PLAN, LC_NCOUNT, LC_NONE, LcError)

__all__ = ["Context", "COUNTER_NAMES", "LC_NONE", "LC_FUSE_ALL", "LC_FUSE_PLAN", "LC_FUSE_APPLY",
           "LC_CORRECT_WINDOW", "LC_CORRECT_ALL", "counts_dict", "camera_struct"]


def counts_dict(arr):
    a = arr.tolist() if hasattr(arr, "tolist") else list(arr)
    return dict(zip(COUNTER_NAMES, [int(x) for x in a]))


def camera_struct(cam) -> _lib.lc_camera:
    d = cam.as_dict() if hasattr(cam, "as_dict") else dict(cam)
    c = _lib.lc_camera()
    c.model = int(d["model"])
    c.fx, c.fy, c.cx, c.cy = float(d["fx"]), float(d["fy"]), float(d["cx"]), float(d["cy"])
    for i in range(4):
        c.k[i] = float(d["k"][i])
    c.min_x, c.max_x = float(d["min_x"]), float(d["max_x"])
    c.min_y, c.max_y = float(d["min_y"]), float(d["max_y"])
    return c


def _params(p) -> _lib.lc_match_params:
    if isinstance(p, _lib.lc_match_params):
        return p
    th, mh, rn, rd, co = p
    return _lib.lc_match_params(int(th), int(mh), int(rn), int(rd), int(co))


_NP = {torch.float32: np.float32, torch.float64: np.float64, torch.int32: np.int32,
       torch.int64: np.int64, torch.uint8: np.uint8, torch.int8: np.int8}


class _Keep:
    """Holds converted arrays alive for the duration of a call."""

    def __init__(self):
        self.refs = []

    def ptr(self, x, dtype=None):
        if x is None:
            return None
        if isinstance(x, torch.Tensor):
            if dtype is not None and _NP.get(x.dtype) != np.dtype(dtype).type:
                x = x.to(dtype={np.float32: torch.float32, np.float64: torch.float64,
                                np.int32: torch.int32, np.int64: torch.int64,
                                np.uint8: torch.uint8, np.int8: torch.int8}[np.dtype(dtype).type])
            x = x.contiguous()
            self.refs.append(x)
            return x.data_ptr()
        a = np.ascontiguousarray(x, dtype=dtype)
        self.refs.append(a)
        return a.ctypes.data


class Graph:
    """A captured sequence of liblc calls (lc_graph_*): launch() replays it on the
    current stream. Holds every buffer the recorded calls reference."""

    def __init__(self, ctx, handle, refs):
        self.ctx, self.h, self.refs = ctx, handle, refs

    def launch(self):
        c = self.ctx
        c._check("lc_graph_launch", c.lib.lc_graph_launch(c.h, self.h, c._stream()))

    def close(self):
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.lc_graph_destroy(self.ctx.h, self.h)
        self.h = None
        self.refs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Capture:
    """`with ctx.capture() as cap: ...` records the liblc calls made inside (on a
    private stream; outputs must be device tensors: host=False) into cap.graph."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.graph = None

    def __enter__(self):
        c = self.ctx
        self.stream = torch.cuda.Stream(device=c.device)
        self.stream.wait_stream(torch.cuda.current_stream(c.device))
        self._sc = torch.cuda.stream(self.stream)
        self._sc.__enter__()
        c._cap_refs = []
        st = c.lib.lc_graph_begin(c.h, c._stream())
        if st != 0:
            c._cap_refs = None
            self._sc.__exit__(None, None, None)
            c._check("lc_graph_begin", st)
        return self

    def __exit__(self, et, ev, tb):
        c = self.ctx
        h = C.c_void_p()
        st = c.lib.lc_graph_end(c.h, c._stream(), C.byref(h))
        refs, c._cap_refs = c._cap_refs, None
        self._sc.__exit__(et, ev, tb)
        torch.cuda.current_stream(c.device).wait_stream(self.stream)
        if et is None:
            c._check("lc_graph_end", st)
            self.graph = Graph(c, h, refs)
        elif st == 0 and h.value:
            c.lib.lc_graph_destroy(c.h, h)
        return False

    def launch(self):
        self.graph.launch()


class Context:
    """One liblc context on one CUDA device (lc_create / lc_destroy)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        self.device = int(device)
        h = C.c_void_p()
        st = self.lib.lc_create(C.byref(h), self.device)
        if st != 0:
            raise LcError("lc_create", st, self.lib.lc_last_error(None).decode())
        self.h = h
        self.n_kf = self.n_feat = self.n_mp = 0
        self.kf_feat_begin = None
        self._cap_refs = None   # buffers referenced by an open capture

    def close(self):
        if getattr(self, "h", None):
            self.lib.lc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing ---------------------------------------------------------------
    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _check(self, fn, st):
        if st != 0:
            raise LcError(fn, st, self.lib.lc_last_error(self.h).decode())

    def _dev(self, n, dtype):
        t = torch.empty(int(n), dtype=dtype, device=f"cuda:{self.device}")
        if self._cap_refs is not None:
            self._cap_refs.append(t)
        return t

    def _keep(self, host):
        """Per-call holder of converted arrays; while capturing, also kept by the graph."""
        if self._cap_refs is not None and host:
            raise LcError("capture", -1, "calls recorded into a graph need host=False")
        k = _Keep()
        if self._cap_refs is not None:
            self._cap_refs.append(k)
        return k

    def capture(self):
        """CUDA-graph capture (lc_graph_begin/end): `with ctx.capture() as cap: ...`,
        then cap.graph.launch() replays the recorded calls."""
        return _Capture(self)

    def kernel_launches(self) -> int:
        return int(self.lib.lc_kernel_launches(self.h))

    def profile_enable(self, on=True):
        self._check("lc_profile_enable", self.lib.lc_profile_enable(self.h, 1 if on else 0))

    def profile_read(self):
        """{family: (device ms, kernel launches)} accumulated since profile_enable()."""
        n = len(_lib.PROF_NAMES)
        ms = (C.c_double * n)()
        la = (C.c_int64 * n)()
        self._check("lc_profile_read", self.lib.lc_profile_read(self.h, ms, la))
        return {name: (ms[i], la[i]) for i, name in enumerate(_lib.PROF_NAMES)}

    def synchronize(self):
        torch.cuda.current_stream(self.device).synchronize()

    # -- lc_upload_map ------------------------------------------------------------
    def upload_map(self, arrays: dict, cams, n_levels=8, scale_factor=1.2, grid=(64, 48), append=False):
        """lc_upload_map: the whole map (REPLACE), or with append=True new keyframes / map
        points after the stored ones (feat_mp / mp_ref_kf in store indices)."""
        k = _Keep()
        a = arrays
        v = _lib.lc_map_view()
        v.n_kf = int(len(a["kf_feat_begin"]) - 1)
        v.n_feat = int(a["feat_mp"].shape[0])
        v.n_mp = int(a["mp_flags"].shape[0])
        spec = dict(kf_pose=np.float64, kf_cam=np.int32, kf_feat_begin=np.int32,
                    feat_uv=np.float32, feat_octave=np.uint8, feat_angle=np.float32,
                    feat_desc=np.uint8, feat_mp=np.int32, mp_pos=np.float32, mp_normal=np.float32,
                    mp_max_dist=np.float32, mp_desc=np.uint8, mp_angle=np.float32,
                    mp_ref_kf=np.int32, mp_flags=np.uint8)
        for name, dt in spec.items():
            setattr(v, name, k.ptr(a[name], dt))
        cams = list(cams) if isinstance(cams, (list, tuple)) else [cams]
        carr = (_lib.lc_camera * len(cams))(*[camera_struct(c) for c in cams])
        prm = _lib.lc_map_params(int(n_levels), int(grid[0]), int(grid[1]), 0, float(scale_factor))
        flags = _lib.LC_UPLOAD_APPEND if append else _lib.LC_UPLOAD_REPLACE
        st = self.lib.lc_upload_map(self.h, C.byref(v), carr, len(cams), C.byref(prm), flags, self._stream())
        self._check("lc_upload_map", st)
        fb = a["kf_feat_begin"]
        fb = (fb.cpu().numpy() if isinstance(fb, torch.Tensor) else np.asarray(fb)).astype(np.int64)
        if append and getattr(self, "kf_feat_begin", None) is not None:
            self.kf_feat_begin = np.r_[self.kf_feat_begin, self.kf_feat_begin[-1] + fb[1:]]
            self.n_kf += v.n_kf
            self.n_feat += v.n_feat
            self.n_mp += v.n_mp
        else:
            self.n_kf, self.n_feat, self.n_mp = v.n_kf, v.n_feat, v.n_mp
            self.kf_feat_begin = fb

    def n_feat_of(self, kfs):
        if self.kf_feat_begin is None:   # no map: the library reports LC_ESTATE
            return 0
        kfs = np.asarray(kfs, np.int64)
        if kfs.size and (kfs.min() < 0 or kfs.max() >= self.n_kf):   # library reports LC_ERANGE
            return 0
        return int(np.sum(self.kf_feat_begin[kfs + 1] - self.kf_feat_begin[kfs]))

    # -- lc_download_map ----------------------------------------------------------
    def download_map(self):
        out = dict(kf_pose=np.zeros((self.n_kf, 13), np.float64),
                   feat_mp=np.zeros(self.n_feat, np.int32),
                   mp_pos=np.zeros((self.n_mp, 3), np.float32),
                   mp_flags=np.zeros(self.n_mp, np.uint8),
                   mp_replaced_by=np.zeros(self.n_mp, np.int32),
                   mp_nobs=np.zeros(self.n_mp, np.int32),
                   mp_normal=np.zeros((self.n_mp, 3), np.float32),
                   mp_max_dist=np.zeros(self.n_mp, np.float32),
                   mp_desc=np.zeros((self.n_mp, 32), np.uint8))
        s = _lib.lc_map_state(*[out[n].ctypes.data for n, _ in _lib.lc_map_state._fields_])
        self._check("lc_download_map", self.lib.lc_download_map(self.h, C.byref(s), self._stream()))
        self.synchronize()
        return out

    def state_save(self):
        self._check("lc_state_save", self.lib.lc_state_save(self.h, self._stream()))

    def state_restore(self):
        self._check("lc_state_restore", self.lib.lc_state_restore(self.h, self._stream()))

    # -- lc_refresh_mappoints -------------------------------------------------------
    def refresh_mappoints(self, mp_idx=None, what=3, host=True):
        """Distinctive descriptor (what & 1) and normal + depth range (what & 2) of the
        given map points (None: all). Returns the counters."""
        k = self._keep(host)
        n = 0 if mp_idx is None else (int(mp_idx.shape[0]) if hasattr(mp_idx, "shape") else len(mp_idx))
        cnt = np.zeros(LC_NCOUNT, np.int64) if host else self._dev(LC_NCOUNT, torch.int64)
        st = self.lib.lc_refresh_mappoints(self.h, n, k.ptr(mp_idx, np.int32), int(what), k.ptr(cnt),
                                           self._stream())
        self._check("lc_refresh_mappoints", st)
        if host:
            self.synchronize()
            return counts_dict(cnt)
        return cnt

    # -- lc_update_connections -----------------------------------------------------
    def update_connections(self, kf_idx=None, th=15, max_edges=64, host=True):
        """Covisibility edges (n_edges [n], kf [n, max_edges], weight [n, max_edges], counts);
        row i is valid up to min(n_edges[i], max_edges), -1 / 0 elsewhere."""
        k = self._keep(host)
        n = self.n_kf if kf_idx is None else (int(kf_idx.shape[0]) if hasattr(kf_idx, "shape") else len(kf_idx))
        if host:
            o_n = np.zeros(n, np.int32)
            o_kf = np.full((n, max_edges), -1, np.int32)
            o_w = np.zeros((n, max_edges), np.int32)
            cnt = np.zeros(LC_NCOUNT, np.int64)
        else:
            o_n = self._dev(n, torch.int32)
            o_kf = self._dev(n * max_edges, torch.int32).fill_(-1)
            o_w = self._dev(n * max_edges, torch.int32).zero_()
            cnt = self._dev(LC_NCOUNT, torch.int64)
        st = self.lib.lc_update_connections(self.h, n if kf_idx is not None else 0, k.ptr(kf_idx, np.int32),
                                            int(th), int(max_edges), k.ptr(o_n), k.ptr(o_kf), k.ptr(o_w),
                                            k.ptr(cnt), self._stream())
        self._check("lc_update_connections", st)
        if host:
            self.synchronize()
            return o_n, o_kf, o_w, counts_dict(cnt)
        return o_n, o_kf.view(n, max_edges), o_w.view(n, max_edges), cnt

    # -- lc_sim3_ransac -------------------------------------------------------------
    def sim3_ransac(self, prob_begin, P1, P2, uv1, uv2, sig1, sig2, cam1, cam2, samples,
                    chi2=9.210, fix_scale=False, refit=True, host=True):
        """Batched Sim3 RANSAC: (S [n_prob, 13], inliers [n_prob], mask [n_corr], counts)."""
        k = self._keep(host)
        pb = np.ascontiguousarray(prob_begin, np.int32)
        n_prob = len(pb) - 1
        n_corr = int(pb[-1]) if n_prob > 0 else 0
        smp = samples if hasattr(samples, "data_ptr") else np.ascontiguousarray(samples, np.int32)
        n_iter = (int(smp.shape[1]) if smp.ndim == 3 else int(smp.shape[0] // max(n_prob, 1) // 3)) if n_prob else 0
        if host:
            S = np.zeros((n_prob, 13), np.float64)
            inl = np.zeros(n_prob, np.int32)
            mask = np.zeros(n_corr, np.uint8)
            cnt = np.zeros(LC_NCOUNT, np.int64)
        else:
            S = self._dev(n_prob * 13, torch.float64)
            inl = self._dev(n_prob, torch.int32)
            mask = self._dev(n_corr, torch.uint8)
            cnt = self._dev(LC_NCOUNT, torch.int64)
        st = self.lib.lc_sim3_ransac(self.h, n_prob, k.ptr(pb), k.ptr(P1, np.float64), k.ptr(P2, np.float64),
                                     k.ptr(uv1, np.float32), k.ptr(uv2, np.float32), k.ptr(sig1, np.float32),
                                     k.ptr(sig2, np.float32), k.ptr(cam1, np.int32), k.ptr(cam2, np.int32),
                                     k.ptr(smp, np.int32), n_iter, float(chi2), int(fix_scale), int(refit),
                                     k.ptr(S), k.ptr(inl), k.ptr(mask), k.ptr(cnt), self._stream())
        self._check("lc_sim3_ransac", st)
        if host:
            self.synchronize()
            return S, inl, mask, counts_dict(cnt)
        return S.view(n_prob, 13), inl, mask, cnt

    def sim3_refine(self, prob_begin, P1, P2, uv1, uv2, sig1, sig2, cam1, cam2, S_init, max_iter=10,
                    th2=10.0, lam=1e-6, host=True):
        """Gauss-Newton Sim3 refinement: (S [n_prob, 13], inliers [n_prob], mask [n_corr], counts)."""
        k = self._keep(host)
        pb = np.ascontiguousarray(prob_begin, np.int32)
        n_prob = len(pb) - 1
        n_corr = int(pb[-1]) if n_prob > 0 else 0
        if host:
            S = np.zeros((n_prob, 13), np.float64)
            inl = np.zeros(n_prob, np.int32)
            mask = np.zeros(n_corr, np.uint8)
            cnt = np.zeros(LC_NCOUNT, np.int64)
        else:
            S = self._dev(n_prob * 13, torch.float64)
            inl = self._dev(n_prob, torch.int32)
            mask = self._dev(n_corr, torch.uint8)
            cnt = self._dev(LC_NCOUNT, torch.int64)
        st = self.lib.lc_sim3_refine(self.h, n_prob, k.ptr(pb), k.ptr(P1, np.float64), k.ptr(P2, np.float64),
                                     k.ptr(uv1, np.float32), k.ptr(uv2, np.float32), k.ptr(sig1, np.float32),
                                     k.ptr(sig2, np.float32), k.ptr(cam1, np.int32), k.ptr(cam2, np.int32),
                                     k.ptr(S_init, np.float64), int(max_iter), float(th2), float(lam),
                                     k.ptr(S), k.ptr(inl), k.ptr(mask), k.ptr(cnt), self._stream())
        self._check("lc_sim3_refine", st)
        if host:
            self.synchronize()
            return S, inl, mask, counts_dict(cnt)
        return S.view(n_prob, 13), inl, mask, cnt

    # -- lc_pgo_sim3 ----------------------------------------------------------------
    def pgo_sim3(self, S_init, fixed, edges, M, max_iter=20, cg_max_iter=500, lambda0=1e-4, eps_dx=1e-8,
                 eps_chi2=1e-10, cg_tol=1e-10, solver="auto", host=True):
        """Essential-graph Sim3 Levenberg-Marquardt: (S [n_v, 13], trace [iters, 6],
        (chi2_0, chi2_final), counts). With host=False S/trace/chi2/counts are device
        tensors (trace [max_iter, 6], counts raw)."""
        k = self._keep(host)
        n_v = int(len(S_init)) if not isinstance(S_init, torch.Tensor) else int(S_init.numel() // 13)
        E = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
        n_e = len(E)
        fx = np.ascontiguousarray(fixed, np.uint8)
        prm = _lib.lc_pgo_params(int(max_iter), int(cg_max_iter), float(lambda0), float(eps_dx),
                                 float(eps_chi2), float(cg_tol), {"auto": 0, "band": 1, "cg": 2, "cr": 3}[solver], 0)
        rows = max(int(max_iter), 1)
        if host:
            S = np.zeros((n_v, 13), np.float64)
            tr = np.zeros((rows, 6), np.float64)
            c2 = np.zeros(2, np.float64)
            cnt = np.zeros(LC_NCOUNT, np.int64)
        else:
            S = self._dev(n_v * 13, torch.float64)
            tr = self._dev(rows * 6, torch.float64)
            c2 = self._dev(2, torch.float64)
            cnt = self._dev(LC_NCOUNT, torch.int64)
        st = self.lib.lc_pgo_sim3(self.h, n_v, k.ptr(S_init, np.float64), k.ptr(fx), n_e, k.ptr(E),
                                  k.ptr(M, np.float64), C.byref(prm), k.ptr(S), k.ptr(tr), k.ptr(c2),
                                  k.ptr(cnt), self._stream())
        self._check("lc_pgo_sim3", st)
        if host:
            self.synchronize()
            cd = counts_dict(cnt)
            return S, tr[:cd["pgo_iters"]], (float(c2[0]), float(c2[1])), cd
        return S.view(n_v, 13), tr.view(rows, 6), c2, cnt

    # -- lc_correct_sim3 ----------------------------------------------------------
    def correct_window(self, cur_kf, S_cw_corr, window, host=True):
        k = self._keep(host)
        window = np.ascontiguousarray(window, np.int32)
        S = np.ascontiguousarray(S_cw_corr, np.float64)
        cur = np.array([int(cur_kf)], np.int32)
        wb = np.array([0, len(window)], np.int32)
        if host:
            outS = np.zeros((len(window), 13), np.float64)
            cnt = np.zeros(LC_NCOUNT, np.int64)
        else:
            outS = self._dev(len(window) * 13, torch.float64)
            cnt = self._dev(LC_NCOUNT, torch.int64)
        st = self.lib.lc_correct_sim3(self.h, LC_CORRECT_WINDOW, 1, k.ptr(cur), k.ptr(S), k.ptr(wb),
                                      k.ptr(window), None, k.ptr(outS), None, None, None, 0, k.ptr(cnt),
                                      self._stream())
        self._check("lc_correct_sim3", st)
        if host:
            self.synchronize()
            return outS, counts_dict(cnt)
        return outS.view(-1, 13), cnt

    def correct_window_batch(self, cur_kf, S_cw_corr, window_begin, window, capacity=None, host=True):
        """LC_CORRECT_WINDOW | LC_DRY_RUN: corrections of several hypotheses, nothing written
        back. Returns (S_corr [sum window, 13], mp_begin [n_batch + 1], mp_idx, mp_pos [n, 3],
        counts)."""
        k = self._keep(host)
        cur = np.ascontiguousarray(cur_kf, np.int32)
        nb = len(cur)
        S = np.ascontiguousarray(S_cw_corr, np.float64).reshape(nb, 13)
        wb = np.ascontiguousarray(window_begin, np.int32)
        win = np.ascontiguousarray(window, np.int32)
        cap = nb * self.n_mp if capacity is None else int(capacity)
        mk = (lambda n, dt, npdt: np.zeros(n, npdt)) if host else (lambda n, dt, npdt: self._dev(n, dt))
        outS = mk(len(win) * 13, torch.float64, np.float64)
        mb = mk(nb + 1, torch.int32, np.int32)
        idx = mk(max(cap, 1), torch.int32, np.int32)
        pos = mk(3 * max(cap, 1), torch.float32, np.float32)
        cnt = mk(LC_NCOUNT, torch.int64, np.int64)
        st = self.lib.lc_correct_sim3(self.h, LC_CORRECT_WINDOW | _lib.LC_DRY_RUN, nb, k.ptr(cur), k.ptr(S),
                                      k.ptr(wb), k.ptr(win), None, k.ptr(outS), k.ptr(mb), k.ptr(idx),
                                      k.ptr(pos), cap, k.ptr(cnt), self._stream())
        self._check("lc_correct_sim3", st)
        if host:
            n = int(mb[-1])
            return outS.reshape(-1, 13), mb, idx[:n], pos.reshape(-1, 3)[:n], counts_dict(cnt)
        return outS.view(-1, 13), mb, idx, pos.view(-1, 3), cnt

    def correct_all(self, S_opt, host=True):
        k = self._keep(host)
        cnt = np.zeros(LC_NCOUNT, np.int64) if host else self._dev(LC_NCOUNT, torch.int64)
        st = self.lib.lc_correct_sim3(self.h, LC_CORRECT_ALL, 0, None, None, None, None,
                                      k.ptr(S_opt, np.float64), None, None, None, None, 0, k.ptr(cnt),
                                      self._stream())
        self._check("lc_correct_sim3", st)
        if host:
            self.synchronize()
            return counts_dict(cnt)
        return cnt

    # -- lc_fuse -------------------------------------------------------------------
    def fuse(self, window, mp_list, params, *, window_S=None, win_list_begin=None,
             phase=LC_FUSE_ALL, w_lo=0, w_hi=None, winner=None, victim=None, action=True,
             debug=False, host=True, cur_kf=-1, forced_mp=None):
        """Returns dict(winner, victim, action, counts[, best, uv, ncand]).
        winner / victim: pass tensors to use them in place (PLAN -> NCCL -> APPLY)."""
        k = self._keep(host)
        window = np.ascontiguousarray(window, np.int32)
        n_w = len(window)
        w_hi = n_w if w_hi is None else int(w_hi)
        if isinstance(win_list_begin, torch.Tensor) and win_list_begin.is_cuda:
            wb = win_list_begin   # device offsets (lc_loop_lists(device=True)); mp_list = its buffer
        else:
            wb = None if win_list_begin is None else np.ascontiguousarray(win_list_begin, np.int32)
        wS = None if window_S is None else (window_S if isinstance(window_S, torch.Tensor)
                                            else np.ascontiguousarray(window_S, np.float64))
        n_list = int(mp_list.shape[0]) if hasattr(mp_list, "shape") else len(mp_list)
        nwf = self.n_feat_of(window)
        nq = (n_list if isinstance(wb, torch.Tensor) else int(wb[-1])) if wb is not None else n_w * n_list
        mk = (lambda n, dt, npdt: np.zeros(n, npdt)) if host else (lambda n, dt, npdt: self._dev(n, dt))
        if winner is None:
            winner = mk(nwf, torch.int64, np.int64)
        if victim is None:
            victim = mk(self.n_mp, torch.int64, np.int64)
        act = mk(nwf, torch.int8, np.int8) if action else None
        cnt = mk(LC_NCOUNT, torch.int64, np.int64)
        dbg = None
        dd = {}
        if debug:
            dd = dict(best=mk(nq, torch.int64, np.int64), uv=mk(2 * nq, torch.float64, np.float64),
                      ncand=mk(nq, torch.int32, np.int32))
            dbg = _lib.lc_query_debug(k.ptr(dd["best"]), k.ptr(dd["uv"]), k.ptr(dd["ncand"]))
        st = self.lib.lc_fuse(self.h, int(phase), int(w_lo), int(w_hi), n_w, k.ptr(window), k.ptr(wS, np.float64),
                              k.ptr(wb), k.ptr(mp_list, np.int32), n_list, C.byref(_params(params)),
                              int(cur_kf), k.ptr(forced_mp, np.int32),
                              k.ptr(winner), k.ptr(victim), k.ptr(act),
                              C.byref(dbg) if dbg is not None else None, k.ptr(cnt), self._stream())
        self._check("lc_fuse", st)
        if host:
            self.synchronize()
        out = dict(winner=winner, victim=victim, action=act,
                   counts=counts_dict(cnt) if host else cnt)
        if debug:
            dd["uv"] = dd["uv"].reshape(-1, 2) if host else dd["uv"].view(-1, 2)
            out.update(dd)
        return out

    # -- lc_loop_lists ---------------------------------------------------------------
    def loop_list_bound(self, src_begin, src_kf):
        """Upper bound of the lists' total length (their source keyframes' features)."""
        fb = self.kf_feat_begin
        sk = np.asarray(src_kf, np.int64)
        return int(np.sum(fb[sk + 1] - fb[sk])) if len(sk) else 0

    def loop_lists(self, src_begin, src_kf, out=None, host=True, device_offsets=False):
        """Loop map-point lists from the resident map: list l = ascending unique map points of
        keyframes src_kf[src_begin[l]:src_begin[l+1]]. Returns (begin [n+1] numpy, lists);
        lists is written into `out` (a device or pinned tensor, >= total entries) if given.
        device_offsets: begin is a device tensor and nothing is read back (no host
        synchronisation); `out` (device) must hold loop_list_bound() entries and is returned
        whole -- pass both to fuse() as mp_list / win_list_begin."""
        k = self._keep(host)
        sb = np.ascontiguousarray(src_begin, np.int32)
        sk = np.ascontiguousarray(src_kf, np.int32)
        n = len(sb) - 1
        if device_offsets:
            ob = self._dev(n + 1, torch.int32)
            if out is None:
                out = self._dev(max(self.loop_list_bound(sb, sk), 1), torch.int32)
            st = self.lib.lc_loop_lists(self.h, n, k.ptr(sb), k.ptr(sk), k.ptr(ob), k.ptr(out), int(out.numel()),
                                        self._stream())
            self._check("lc_loop_lists", st)
            return ob, out
        ob = np.zeros(n + 1, np.int32)
        if out is None:
            fb = self.kf_feat_begin
            ok = sk[(sk >= 0) & (sk < len(fb) - 1)]   # (out-of-range ids: the library reports LC_ERANGE)
            cap = int(np.sum(fb[ok + 1] - fb[ok])) if len(ok) else 0
            out = np.zeros(max(cap, 1), np.int32) if host else self._dev(max(cap, 1), torch.int32)
        cap = int(out.numel() if isinstance(out, torch.Tensor) else out.size)
        st = self.lib.lc_loop_lists(self.h, n, k.ptr(sb), k.ptr(sk), k.ptr(ob), k.ptr(out), cap, self._stream())
        self._check("lc_loop_lists", st)
        return ob, out[:int(ob[-1])]

    # -- lc_fuse_adds (sparse ADD exchange of a sharded fusion) --------------------
    def fuse_adds_pack(self, window, w_lo, w_hi, winner, idx, word):
        """Compact the shard's winner words on empty slots into (idx, word); returns n."""
        k = self._keep(False)
        window = np.ascontiguousarray(window, np.int32)
        n = C.c_int64(0)
        st = self.lib.lc_fuse_adds(self.h, _lib.LC_ADDS_PACK, len(window), k.ptr(window), int(w_lo), int(w_hi),
                                   k.ptr(winner), k.ptr(idx), k.ptr(word), C.byref(n), int(idx.numel()),
                                   self._stream())
        self._check("lc_fuse_adds", st)
        return int(n.value)

    def fuse_adds_unpack(self, window, winner, idx, word):
        """winner <- NONE, winner[idx] = word (the dense table APPLY reads)."""
        k = self._keep(False)
        window = np.ascontiguousarray(window, np.int32)
        n = C.c_int64(int(idx.numel()))
        idx = idx.contiguous()
        word = word.contiguous()
        st = self.lib.lc_fuse_adds(self.h, _lib.LC_ADDS_UNPACK, len(window), k.ptr(window), 0, len(window),
                                   k.ptr(winner), k.ptr(idx) if idx.numel() else None,
                                   k.ptr(word) if word.numel() else None, C.byref(n), int(idx.numel()),
                                   self._stream())
        self._check("lc_fuse_adds", st)

    # -- lc_set_point_range / lc_mp_positions (sharded correction) -------------------
    def set_point_range(self, lo=0, hi=-1):
        """Later WINDOW / ALL corrections rewrite the positions of map points [lo, hi) only
        (hi < 0: all); poses, owners and corr_ref stay replicated."""
        self._check("lc_set_point_range", self.lib.lc_set_point_range(self.h, int(lo), int(hi)))

    def mp_positions(self, op, lo, hi, xyz=None, host=True):
        """LC_POS_GET: fp32 positions of map points [lo, hi) into xyz (new if None);
        LC_POS_SET: xyz [hi - lo][3] into the store. Returns xyz."""
        k = self._keep(host)
        n = max(int(hi) - int(lo), 0)
        if xyz is None:
            xyz = np.zeros((n, 3), np.float32) if host else self._dev(3 * n, torch.float32).view(n, 3)
        st = self.lib.lc_mp_positions(self.h, int(op), int(lo), int(hi), k.ptr(xyz) if n else None, self._stream())
        self._check("lc_mp_positions", st)
        if host and op == _lib.LC_POS_GET:
            self.synchronize()
        return xyz

    # -- lc_search_by_projection ----------------------------------------------------
    def search_by_projection(self, pair_kf, pair_S, pair_param, params, pair_list_begin, mp_list,
                             pair_taken=None, debug=False, host=True):
        k = self._keep(host)
        pair_kf = np.ascontiguousarray(pair_kf, np.int32)
        n_pairs = len(pair_kf)
        plb = np.ascontiguousarray(pair_list_begin, np.int32)
        prms = (_lib.lc_match_params * len(params))(*[_params(p) for p in params])
        ntot = self.n_feat_of(pair_kf)
        nq = int(plb[-1])
        mk = (lambda n, dt, npdt: np.zeros(n, npdt)) if host else (lambda n, dt, npdt: self._dev(n, dt))
        o_mp = mk(ntot, torch.int32, np.int32)
        o_d = mk(ntot, torch.int32, np.int32)
        cnt = mk(n_pairs * LC_NCOUNT, torch.int64, np.int64)
        dbg = None
        dd = {}
        if debug:
            dd = dict(best=mk(nq, torch.int64, np.int64), uv=mk(2 * nq, torch.float64, np.float64),
                      ncand=mk(nq, torch.int32, np.int32))
            dbg = _lib.lc_query_debug(k.ptr(dd["best"]), k.ptr(dd["uv"]), k.ptr(dd["ncand"]))
        st = self.lib.lc_search_by_projection(
            self.h, n_pairs, k.ptr(pair_kf), k.ptr(pair_S, np.float64), k.ptr(pair_param, np.int32),
            prms, len(params), k.ptr(plb), k.ptr(mp_list, np.int32), k.ptr(pair_taken, np.int32),
            k.ptr(o_mp), k.ptr(o_d), C.byref(dbg) if dbg is not None else None, k.ptr(cnt),
            self._stream())
        self._check("lc_search_by_projection", st)
        if host:
            self.synchronize()
            cnt = cnt.reshape(n_pairs, LC_NCOUNT)
        else:
            cnt = cnt.view(n_pairs, LC_NCOUNT)
        out = dict(feat_mp=o_mp, feat_dist=o_d, counts=cnt)
        if debug:
            dd["uv"] = dd["uv"].reshape(-1, 2) if host else dd["uv"].view(-1, 2)
            out.update(dd)
        return out
