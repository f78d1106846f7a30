# PGO cyclic-reduction solver: parity tests + C3/C5 timing (auto = CR vs band)
set -x
timeout 900 python -m pytest tests/test_gpu_pgo.py -m gpu -q -x 2>&1 | tail -6
timeout 300 python - <<'PY'
import time, numpy as np, torch
from paper_2603_17201_b200 import Context
from lcsynth import make_pose_graph
c = Context(0)
for name in ("C2", "C3", "C5"):
    g = make_pose_graph(name, 0)
    gS, gM = torch.from_numpy(g.S_init).cuda(), torch.from_numpy(g.M).cuda()
    for solver in ("auto", "band"):
        ts = []
        for i in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); r = c.pgo_sim3(gS, g.fixed, g.edges, gM, max_iter=20, host=False, solver=solver); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        cnt = r[3].cpu().numpy()
        print(name, solver, "ms", [round(t, 2) for t in ts], "iters", cnt[32], "band", cnt[36], "cr_levels", cnt[39], "chi2", r[2].cpu().numpy())
PY
