"""FUSE_ALL determinism probe: the same loop event N times; post-apply feat_mp / n_obs must agree."""
import sys
import numpy as np
sys.path.insert(0, ".")
from lcsynth import make_world
from lcsynth.world import FUSE_PARAMS
from paper_2603_17201_b200 import Context
name = sys.argv[1] if len(sys.argv) > 1 else "S3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = make_world(name, 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
ctx.state_save()
res = []
for i in range(n):
    ctx.state_restore()
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    g = ctx.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
    st = ctx.download_map()
    res.append((st["feat_mp"].copy(), st["mp_nobs"].copy(), g["counts"]))
for i in range(1, n):
    d = np.nonzero(res[i][0] != res[0][0])[0]
    print(name, i, "feat_mp diffs", len(d), d[:10], res[0][0][d[:10]], res[i][0][d[:10]],
          "nobs diffs", int(np.sum(res[i][1] != res[0][1])))
print("counts", {k: v for k, v in res[0][2].items() if k in ("rewired", "dup_cleared", "added")})
