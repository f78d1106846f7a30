"""Device-offset loop-list build at C5: event time per call (run under ncu for per-kernel times)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
from lcsynth import make_world
from paper_2603_17201_b200 import Context
w = make_world("C5", 0)
ctx = Context(0)
ctx.upload_map(w.map_arrays(), [w.cam])
dev = torch.device("cuda:0")
out = torch.empty(ctx.loop_list_bound(w.list_src_begin, w.list_src_kf), dtype=torch.int32, device=dev)
sb = torch.from_numpy(w.list_src_begin).pin_memory(); sk = torch.from_numpy(w.list_src_kf).pin_memory()
st = torch.cuda.current_stream()
for i in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(st)
    ob, l = ctx.loop_lists(sb, sk, out=out, host=False, device_offsets=True)
    b.record(st); b.synchronize()
    if i >= 2: print(f"lists (device offsets): {a.elapsed_time(b):.3f} ms")
