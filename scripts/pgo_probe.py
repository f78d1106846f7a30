"""Time lc_pgo_sim3 on the synthetic essential graphs (CUDA events on the call stream)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from lcsynth import make_pose_graph  # noqa: E402
from paper_2603_17201_b200 import Context  # noqa: E402

ctx = Context(0)
for name in sys.argv[1:] or ["C2", "C3", "C5"]:
    g = make_pose_graph(name, 0)
    S0 = torch.from_numpy(g.S_init).cuda()
    M = torch.from_numpy(g.M).cuda()
    for solver, cg_tol in (("auto", 1e-10), ("cg", 1e-10)):
        ctx.pgo_sim3(S0, g.fixed, g.edges, M, host=False, cg_tol=cg_tol, solver=solver)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(3):
            a.record()
            S, tr, c2, cnt = ctx.pgo_sim3(S0, g.fixed, g.edges, M, host=False, cg_tol=cg_tol, solver=solver)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        from paper_2603_17201_b200 import COUNTER_NAMES
        cd = dict(zip(COUNTER_NAMES, cnt.cpu().numpy().tolist()))
        c2 = c2.cpu().numpy()
        tr = tr.cpu().numpy()[:cd["pgo_iters"]]
        print(f"{name} n_v={g.n_v} n_e={g.n_e} {solver} cg_tol={cg_tol:g} ms={np.median(ms):.3f} iters={cd['pgo_iters']} "
              f"acc={cd['pgo_accepted']} solver_it={cd['pgo_solver_iters']} stop={cd['pgo_stop']} bw={cd['pgo_band'] - 1} chi2 {c2[0]:.6g}->{c2[1]:.6g}", flush=True)
        print("   cg per iter", tr[:, 5].astype(int).tolist())
ctx.close()
