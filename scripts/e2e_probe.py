"""Per-call breakdown of bench.py's e2e step at C5 (events + host wall clock per call)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from lcsynth import make_world
from lcsynth.world import FUSE_PARAMS
from paper_2603_17201_b200 import Context

w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
ctx.state_save()
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
n_wfeat = ctx.n_feat_of(w.window)
tables = torch.empty(n_wfeat + w.n_mp, dtype=torch.int64, device=dev)
win_t, vic_t = tables[:n_wfeat], tables[n_wfeat:]
Sopt_pin = torch.from_numpy(w.S_opt).pin_memory()
winS_pin = torch.from_numpy(np.ascontiguousarray(w.win_S)).pin_memory()
winS_dev = winS_pin.to(dev)
sb_pin = torch.from_numpy(w.list_src_begin).pin_memory()
sk_pin = torch.from_numpy(w.list_src_kf).pin_memory()
lst_dev = torch.empty(len(w.mp_list) + 1024, dtype=torch.int32, device=dev)
cnt_pin = torch.empty(64, dtype=torch.int64).pin_memory()


def timed(name, fn, rec):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(st)
    r = fn()
    b.record(st)
    t1 = time.perf_counter()
    b.synchronize()
    t2 = time.perf_counter()
    rec.setdefault(name, []).append((a.elapsed_time(b), 1e3 * (t1 - t0), 1e3 * (t2 - t0)))
    return r


for variant in ("pinned winS", "device winS"):
    rec = {}
    for i in range(8):
        ctx.state_restore()
        torch.cuda.synchronize()
        lb, lst = timed("loop_lists", lambda: ctx.loop_lists(sb_pin, sk_pin, out=lst_dev, host=False), rec)
        timed("correct_window", lambda: ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window, host=False), rec)
        ws_ = winS_pin if variant == "pinned winS" else winS_dev
        r = timed("fuse", lambda: ctx.fuse(w.window, lst, FUSE_PARAMS, window_S=ws_, win_list_begin=lb,
                                           winner=win_t, victim=vic_t, action=False, host=False), rec)
        timed("correct_all", lambda: ctx.correct_all(Sopt_pin, host=False), rec)
    print("==", variant)
    for k, v in rec.items():
        v = np.array(v[3:])
        print(f"  {k:15s} events {v[:,0].mean():8.3f} ms  enqueue {v[:,1].mean():8.3f} ms  wall {v[:,2].mean():8.3f} ms")
