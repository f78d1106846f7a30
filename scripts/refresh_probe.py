"""One C5 loop event + refresh of the loop's points (for ncu)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from lcsynth import make_world
from lcsynth.world import FUSE_PARAMS
from paper_2603_17201_b200 import Context

w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
ctx.fuse(w.window, torch.from_numpy(w.mp_list).cuda(), FUSE_PARAMS, window_S=w.win_S,
         win_list_begin=w.win_list_begin)
sel = torch.from_numpy(np.unique(w.mp_list).astype(np.int32)).cuda()
print(ctx.refresh_mappoints(sel, what=3))
n, kf, w, c = ctx.update_connections(None, th=15, max_edges=64)
print(c["conn_kf"], c["conn_edges"], int(n.max()))
