"""cProfile of the Python side of lc_fuse calls (host enqueue analysis)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS  # noqa: E402
from paper_2603_17201_b200 import Context  # noqa: E402

w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
ctx.state_save()
dev = torch.device("cuda:0")
lst = torch.from_numpy(w.mp_list).to(dev)
win = torch.empty(ctx.n_feat_of(w.window), dtype=torch.int64, device=dev)
vic = torch.empty(w.n_mp, dtype=torch.int64, device=dev)


def go():
    for _ in range(20):
        ctx.fuse(w.window, lst, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin, winner=win,
                 victim=vic, action=False, host=False)
        torch.cuda.synchronize()


go()
pr = cProfile.Profile()
pr.enable()
go()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
