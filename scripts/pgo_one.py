"""One lc_pgo_sim3 call on a named graph (ncu target): python scripts/pgo_one.py C2 cr 20"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2603_17201_b200 import Context  # noqa: E402
from lcsynth import make_pose_graph  # noqa: E402
name, solver, it = sys.argv[1], sys.argv[2], int(sys.argv[3])
c = Context(0)
g = make_pose_graph(name, 0)
r = c.pgo_sim3(torch.from_numpy(g.S_init).cuda(), g.fixed, g.edges, torch.from_numpy(g.M).cuda(), max_iter=it,
               host=False, solver=solver)
torch.cuda.synchronize()
cnt = r[3].cpu().numpy()
print(cnt[32:40], 'timing', cnt[:8], 'elim', cnt[8:13])
