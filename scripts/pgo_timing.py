"""Per-phase cycles of the banded PGO solve (needs a -DLC_PGO_TIMING=1 build via LC_LIB_PATH)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from lcsynth import make_pose_graph  # noqa: E402
from paper_2603_17201_b200 import Context  # noqa: E402

ctx = Context(0)
for name in sys.argv[1:] or ["C2", "C5"]:
    g = make_pose_graph(name, 0)
    S, tr, c2, cnt = ctx.pgo_sim3(g.S_init, g.fixed, g.edges, g.M, solver="band", host=False)
    c = cnt.cpu().numpy().astype(np.float64)
    npos = c[6]
    print(name, "cycles per position: chol+y %.0f panel %.0f update %.0f retire %.0f load %.0f | backsub total %.0f"
          % tuple(c[:6] / npos), flush=True)
ctx.close()
