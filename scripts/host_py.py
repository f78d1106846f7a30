"""Python vs C++ share of the host cost of lc_fuse (C5 loop event)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS  # noqa: E402
from paper_2603_17201_b200 import Context, lc  # noqa: E402

w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
dev = torch.device("cuda:0")
lst = torch.from_numpy(w.mp_list).to(dev)
win = torch.empty(ctx.n_feat_of(w.window), dtype=torch.int64, device=dev)
vic = torch.empty(w.n_mp, dtype=torch.int64, device=dev)
orig = ctx.lib.lc_fuse
acc = []


def timed(*a):
    t = time.perf_counter()
    r = orig(*a)
    acc.append(time.perf_counter() - t)
    return r


class L:
    def __getattr__(self, n):
        return timed if n == "lc_fuse" else getattr(ctx.__dict__["_L"], n)


ctx._L = ctx.lib
ctx.lib = L()
tt = []
for i in range(25):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx.fuse(w.window, lst, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin, winner=win, victim=vic,
             action=False, host=False)
    tt.append(time.perf_counter() - t)
print(f"fuse wrapper {1e6 * np.median(tt[5:]):.1f} us, of which the C call {1e6 * np.median(acc[5:]):.1f} us")
t = time.perf_counter()
for i in range(20):
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window, host=False)
torch.cuda.synchronize()
print(f"correct_window wrapper {1e6 * (time.perf_counter() - t) / 20:.1f} us (incl. GPU)")
