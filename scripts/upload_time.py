import sys, time
import torch
sys.path.insert(0, ".")
from lcsynth import make_world
from paper_2603_17201_b200 import Context
w = make_world("C5", 0)
arr = w.map_arrays()
pin = {k: torch.from_numpy(v.copy() if hasattr(v, "copy") else v).pin_memory() for k, v in arr.items()}
for label, a in (("pageable", arr), ("pinned", pin), ("pageable", arr)):
    ctx = Context(0)
    torch.cuda.synchronize(); t = time.perf_counter()
    ctx.upload_map(a, [w.cam]); torch.cuda.synchronize()
    print(label, f"{1e3 * (time.perf_counter() - t):.1f} ms")
    ctx.close()
