"""ctypes declarations of include/lc.h (argument marshalling only).

Loads the in-tree liblc.so and fails loudly when it is missing: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LC_LIB_PATH") or os.path.join(PKG, "liblc.so")

LC_OK, LC_EINVAL, LC_ESTATE, LC_ECUDA, LC_ENOMEM, LC_ERANGE, LC_ECAPACITY = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "LC_OK", -1: "LC_EINVAL", -2: "LC_ESTATE", -3: "LC_ECUDA", -4: "LC_ENOMEM",
                -5: "LC_ERANGE", -6: "LC_ECAPACITY"}
LC_NONE = (1 << 63) - 1
LC_CORRECT_WINDOW, LC_CORRECT_ALL, LC_DRY_RUN = 1, 2, 4
LC_FUSE_PLAN, LC_FUSE_APPLY, LC_FUSE_ALL = 1, 2, 3
LC_ADDS_PACK, LC_ADDS_UNPACK = 1, 2
LC_POS_GET, LC_POS_SET = 1, 2
LC_UPLOAD_REPLACE, LC_UPLOAD_APPEND = 0, 1
LC_REFRESH_DESC, LC_REFRESH_NORMAL = 1, 2
COUNTER_NAMES = [
    "queries", "skip_bad", "skip_found", "cull_depth", "cull_bounds", "cull_dist",
    "cull_angle", "candidates", "no_cand", "over_th", "ratio_rej", "proposals",
    "winners", "orient_rej", "add", "victim_prop", "loop_skip", "bad_slot",
    "victims", "rewired", "dup_cleared", "added", "corr_kf", "corr_mp",
    "refresh_mp", "refresh_obs", "conn_kf", "conn_edges", "ransac_hyp", "ransac_inliers",
    "refine_iters", "refine_inliers", "pgo_iters", "pgo_accepted", "pgo_solver_iters", "pgo_stop",
    "pgo_band", "forced", "edge_amb", "pgo_cr_levels",
]
LC_NCOUNT = len(COUNTER_NAMES)
PROF_NAMES = ["upload", "correct_window", "correct_all", "fuse_prep", "match", "resolve", "apply",
              "sbp_match", "sbp_resolve", "state", "project", "refresh", "conn", "ransac", "refine", "pgo"]


class lc_sim3(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("s", C.c_double)]


class lc_camera(C.Structure):
    _fields_ = [("model", C.c_int32), ("reserved", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double), ("k", C.c_double * 4),
                ("min_x", C.c_double), ("max_x", C.c_double), ("min_y", C.c_double),
                ("max_y", C.c_double)]


class lc_map_params(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("grid_cols", C.c_int32), ("grid_rows", C.c_int32),
                ("reserved", C.c_int32), ("scale_factor", C.c_double)]


class lc_map_view(C.Structure):
    _fields_ = [("n_kf", C.c_int32), ("n_feat", C.c_int32), ("n_mp", C.c_int32),
                ("reserved", C.c_int32)] + [
        (n, C.c_void_p) for n in ("kf_pose", "kf_cam", "kf_feat_begin", "feat_uv", "feat_octave",
                                  "feat_angle", "feat_desc", "feat_mp", "mp_pos", "mp_normal",
                                  "mp_max_dist", "mp_desc", "mp_angle", "mp_ref_kf", "mp_flags")]


class lc_map_state(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("kf_pose", "feat_mp", "mp_pos", "mp_flags",
                                          "mp_replaced_by", "mp_nobs", "mp_normal",
                                          "mp_max_dist", "mp_desc")]


class lc_match_params(C.Structure):
    _fields_ = [("th", C.c_int32), ("max_hamming", C.c_int32), ("ratio_num", C.c_int32),
                ("ratio_den", C.c_int32), ("check_orientation", C.c_int32)]


class lc_query_debug(C.Structure):
    _fields_ = [("best", C.c_void_p), ("uv", C.c_void_p), ("ncand", C.c_void_p)]


class lc_pgo_params(C.Structure):
    _fields_ = [("max_iter", C.c_int32), ("cg_max_iter", C.c_int32), ("lambda0", C.c_double),
                ("eps_dx", C.c_double), ("eps_chi2", C.c_double), ("cg_tol", C.c_double),
                ("solver", C.c_int32), ("reserved", C.c_int32)]


class LcError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__(f"{fn} failed: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load():
    """Load liblc.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"liblc.so not found at {LIB_PATH}; run paper_2603_17201_b200/build.py "
                           "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    P = C.POINTER
    sig = {
        "lc_create": (i32, [P(vp), i32]),
        "lc_destroy": (i32, [vp]),
        "lc_last_error": (C.c_char_p, [vp]),
        "lc_kernel_launches": (i64, [vp]),
        "lc_profile_enable": (i32, [vp, i32]),
        "lc_profile_read": (i32, [vp, vp, vp]),
        "lc_upload_map": (i32, [vp, P(lc_map_view), vp, i32, P(lc_map_params), i32, vp]),
        "lc_download_map": (i32, [vp, P(lc_map_state), vp]),
        "lc_state_save": (i32, [vp, vp]),
        "lc_state_restore": (i32, [vp, vp]),
        "lc_correct_sim3": (i32, [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp]),
        "lc_fuse": (i32, [vp, i32, i32, i32, i32, vp, vp, vp, vp, i64, P(lc_match_params), i32, vp, vp,
                          vp, vp, vp, vp, vp]),
        "lc_loop_lists": (i32, [vp, i32, vp, vp, vp, vp, i64, vp]),
        "lc_fuse_adds": (i32, [vp, i32, i32, vp, i32, i32, vp, vp, vp, vp, i64, vp]),
        "lc_set_point_range": (i32, [vp, i32, i32]),
        "lc_mp_positions": (i32, [vp, i32, i32, i32, vp, vp]),
        "lc_search_by_projection": (i32, [vp, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp,
                                          vp, vp]),
        "lc_refresh_mappoints": (i32, [vp, i32, vp, i32, vp, vp]),
        "lc_update_connections": (i32, [vp, i32, vp, i32, i32, vp, vp, vp, vp, vp]),
        "lc_sim3_ransac": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, C.c_double, i32,
                                 i32, vp, vp, vp, vp, vp]),
        "lc_sim3_refine": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, C.c_double,
                                 C.c_double, vp, vp, vp, vp, vp]),
        "lc_pgo_sim3": (i32, [vp, i32, vp, vp, i32, vp, vp, P(lc_pgo_params), vp, vp, vp, vp, vp]),
        "lc_graph_begin": (i32, [vp, vp]),
        "lc_graph_end": (i32, [vp, vp, P(vp)]),
        "lc_graph_launch": (i32, [vp, vp, vp]),
        "lc_graph_destroy": (i32, [vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return ["lc_create", "lc_destroy", "lc_last_error", "lc_kernel_launches", "lc_profile_enable",
            "lc_profile_read", "lc_upload_map",
            "lc_download_map", "lc_state_save", "lc_state_restore", "lc_correct_sim3", "lc_fuse", "lc_fuse_adds", "lc_loop_lists",
            "lc_set_point_range", "lc_mp_positions",
            "lc_search_by_projection", "lc_refresh_mappoints", "lc_update_connections", "lc_sim3_ransac", "lc_sim3_refine", "lc_pgo_sim3", "lc_graph_begin", "lc_graph_end", "lc_graph_launch",
            "lc_graph_destroy"]
