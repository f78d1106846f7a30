"""One C5 loop event, then lc_refresh_mappoints and lc_update_connections (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS  # noqa: E402
from paper_2603_17201_b200 import Context  # noqa: E402

w = make_world("C5", 0)
c = Context(0)
c.upload_map(w.map_arrays(), [w.cam])
c.correct_window(w.cur_kf, w.S_cw_corr, w.window)
c.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
mp = np.unique(w.mp_list).astype(np.int32)
for _ in range(2):
    c.refresh_mappoints(mp)
    c.update_connections(None, th=15)
torch.cuda.synchronize()
print("ok")
