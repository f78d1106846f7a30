"""bench.py's e2e step repeated 40 times: per-step event ms and per-call host enqueue ms (spike hunt)."""
import sys, time, gc
import numpy as np, torch
sys.path.insert(0, ".")
from lcsynth import make_world
from lcsynth.world import FUSE_PARAMS
from paper_2603_17201_b200 import Context
w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
ctx.state_save()
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
n_wfeat = ctx.n_feat_of(w.window)
tables = torch.empty(n_wfeat + w.n_mp, dtype=torch.int64, device=dev)
win_t, vic_t = tables[:n_wfeat], tables[n_wfeat:]
Sopt_pin = torch.from_numpy(w.S_opt).pin_memory()
winS_pin = torch.from_numpy(np.ascontiguousarray(w.win_S)).pin_memory()
sb_pin = torch.from_numpy(w.list_src_begin).pin_memory(); sk_pin = torch.from_numpy(w.list_src_kf).pin_memory()
cnt_pin = torch.empty(64, dtype=torch.int64).pin_memory()
lst_dev = torch.empty(len(w.mp_list) + 1024, dtype=torch.int32, device=dev)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
gcoff = len(sys.argv) > 1 and sys.argv[1] == "nogc"
if gcoff: gc.disable()
for i in range(40):
    ctx.state_restore(); flush.fill_(1.0); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = [time.perf_counter()]
    a.record(st)
    lb, lst = ctx.loop_lists(sb_pin, sk_pin, out=lst_dev, host=False); t.append(time.perf_counter())
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window, host=False); t.append(time.perf_counter())
    r = ctx.fuse(w.window, lst, FUSE_PARAMS, window_S=winS_pin, win_list_begin=lb, winner=win_t, victim=vic_t,
                 action=False, host=False); t.append(time.perf_counter())
    ctx.correct_all(Sopt_pin, host=False); t.append(time.perf_counter())
    cnt_pin[:r["counts"].numel()].copy_(r["counts"], non_blocking=True)
    b.record(st); b.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"{i:2d} ev {a.elapsed_time(b):7.3f} ms | lists {d[0]:6.3f} win {d[1]:6.3f} fuse {d[2]:6.3f} all {d[3]:6.3f} sync {d[4]:6.3f}")
