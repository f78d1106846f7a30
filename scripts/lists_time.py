import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from lcsynth import make_world
from paper_2603_17201_b200 import Context
w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
dev = torch.device("cuda:0")
out = torch.empty(len(w.mp_list) + 1024, dtype=torch.int32, device=dev)
sb = torch.from_numpy(w.list_src_begin).pin_memory(); sk = torch.from_numpy(w.list_src_kf).pin_memory()
st = torch.cuda.current_stream()
for i in range(8):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(st)
    lb, l = ctx.loop_lists(sb, sk, out=out, host=False)
    b.record(st); b.synchronize(); t1 = time.perf_counter()
    if i >= 3: print(f"lists: events {a.elapsed_time(b):.3f} ms, wall {1e3*(t1-t0):.3f} ms")
pin = torch.from_numpy(w.mp_list).pin_memory(); d = torch.empty_like(pin, device=dev)
for i in range(3):
    torch.cuda.synchronize(); a.record(st); d.copy_(pin, non_blocking=True); b.record(st); b.synchronize()
print(f"H2D of the lists ({pin.numel()*4/1e6:.1f} MB): {a.elapsed_time(b):.3f} ms")
