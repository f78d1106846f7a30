"""Is the eager C5 step host-bound on this box? Per step: CUDA-event time (as bench.py),
host enqueue time of step(), and the same step timed after a full sync."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from lcsynth import make_world
from lcsynth.world import FUSE_PARAMS
from paper_2603_17201_b200 import Context
w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam]); ctx.state_save()
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
mp_list_d = torch.from_numpy(w.mp_list).to(dev)
win_S_d = torch.from_numpy(np.ascontiguousarray(w.win_S)).to(dev)
S_opt_d = torch.from_numpy(w.S_opt).to(dev)
n_wfeat = ctx.n_feat_of(w.window)
tables = torch.empty(n_wfeat + w.n_mp, dtype=torch.int64, device=dev)
win_t, vic_t = tables[:n_wfeat], tables[n_wfeat:]
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
def step():
    t = [time.perf_counter()]
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window, host=False); t.append(time.perf_counter())
    ctx.fuse(w.window, mp_list_d, FUSE_PARAMS, window_S=win_S_d, win_list_begin=w.win_list_begin, winner=win_t,
             victim=vic_t, action=False, host=False); t.append(time.perf_counter())
    ctx.correct_all(S_opt_d, host=False); t.append(time.perf_counter())
    return np.diff(t) * 1e3
for mode in ("bench", "synced"):
    rows = []
    for i in range(13):
        ctx.state_restore(); flush.fill_(1.0)
        if mode == "synced": torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); h = step(); b.record(st)
        rows.append((a, b, h))
    torch.cuda.synchronize()
    ev = np.array([a.elapsed_time(b) for a, b, _ in rows[3:]])
    hs = np.array([h for _, _, h in rows[3:]])
    print(mode, "event ms mean %.4f min %.4f max %.4f | host ms win %.3f fuse %.3f all %.3f" %
          (ev.mean(), ev.min(), ev.max(), *hs.mean(0)))
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)
print(subprocess.run(["bash", "-c", "nproc; uptime; lscpu | grep 'Model name'"], capture_output=True, text=True).stdout)
