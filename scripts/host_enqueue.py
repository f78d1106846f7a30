"""Host-side enqueue time of one C5 loop event (the three API calls, no synchronisation)
against its device time: is the eager step host-bound?"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS  # noqa: E402
from paper_2603_17201_b200 import Context  # noqa: E402

w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
ctx.state_save()
dev = torch.device("cuda:0")
lst = torch.from_numpy(w.mp_list).to(dev)
Sop = torch.from_numpy(w.S_opt).to(dev)
n_wfeat = ctx.n_feat_of(w.window)
win = torch.empty(n_wfeat, dtype=torch.int64, device=dev)
vic = torch.empty(w.n_mp, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream()
res = []
for i in range(12):
    ctx.state_restore()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    t0 = time.perf_counter()
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window, host=False)
    t1 = time.perf_counter()
    ctx.fuse(w.window, lst, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin, winner=win, victim=vic,
             action=False, host=False)
    t2 = time.perf_counter()
    ctx.correct_all(Sop, host=False)
    t3 = time.perf_counter()
    b.record(st)
    b.synchronize()
    if i >= 2:
        res.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), a.elapsed_time(b)))
r = np.array(res).mean(0)
print(f"host enqueue ms: window {r[0]:.3f} fuse {r[1]:.3f} all {r[2]:.3f} total {r[:3].sum():.3f} | device step {r[3]:.3f}")
