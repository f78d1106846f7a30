"""Keyframe-sharded fusion (paper_2603_17201_b200/dist.py) with real liblc contexts:
two ranks (gloo, both on cuda:0 -- the GPU box has one device) run PLAN on their shard,
merge the victim words by all_reduce(MIN), exchange the sparse ADD lists (lc_fuse_adds)
and APPLY; the gathered tables and the final map store must equal single-GPU FUSE_ALL bit
for bit (readings A17, A21). The NCCL
launch of bench.py runs the same code with one device per rank."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from lcsynth import make_world  # noqa: E402
from lcsynth.world import FUSE_PARAMS  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, on_device, out_path):
    import torch.distributed as dist
    from paper_2603_17201_b200 import Context
    from paper_2603_17201_b200.dist import correct_all_sharded, correct_window_sharded, fuse_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = make_world(name, 0)
    ctx = Context(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    dev = torch.device("cuda:0") if on_device else None
    # the whole loop event sharded: WINDOW and ALL point passes by map-point
    # slice + position all_gather, the fuse by keyframe shard + victim MIN + ADD gather
    cw, _ = correct_window_sharded(ctx, w.cur_kf, w.S_cw_corr, w.window, device=dev)
    lst = torch.from_numpy(w.mp_list).cuda() if on_device else w.mp_list
    pc, ac, info = fuse_sharded(ctx, w.window, lst, FUSE_PARAMS, window_S=w.win_S,
                                win_list_begin=w.win_list_begin, device=dev, gather_winner=True)
    S_opt = torch.from_numpy(w.S_opt).cuda() if on_device else w.S_opt
    ca, _ = correct_all_sharded(ctx, S_opt, device=dev)
    torch.cuda.synchronize()
    st = ctx.download_map()
    np.savez(f"{out_path}.{rank}.npz", winner=info["winner"].cpu().numpy(), victim=info["victim"].cpu().numpy(),
             feat_mp=st["feat_mp"], mp_flags=st["mp_flags"], mp_replaced_by=st["mp_replaced_by"],
             mp_nobs=st["mp_nobs"], mp_pos=st["mp_pos"], kf_pose=st["kf_pose"])
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["T5", "C2", "S3"])
@pytest.mark.parametrize("on_device", [False, True], ids=["host-tables", "device-tables"])
def test_sharded_fuse_two_ranks_equals_single_gpu(tmp_path, name, on_device):
    import torch.multiprocessing as mp
    from paper_2603_17201_b200 import Context, build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "r")
    mp.start_processes(_worker, args=(2, _free_port(), name, on_device, out), nprocs=2, join=True,
                       start_method="spawn")
    w = make_world(name, 0)
    ctx = Context(0)
    ctx.upload_map(w.map_arrays(), [w.cam])
    ctx.correct_window(w.cur_kf, w.S_cw_corr, w.window)
    g = ctx.fuse(w.window, w.mp_list, FUSE_PARAMS, window_S=w.win_S, win_list_begin=w.win_list_begin)
    ctx.correct_all(w.S_opt)
    st = ctx.download_map()
    for r in range(2):
        d = np.load(f"{out}.{r}.npz")
        assert np.array_equal(d["winner"], g["winner"]), f"rank {r}: gathered winner table"
        assert np.array_equal(d["victim"], g["victim"]), f"rank {r}: merged victim table"
        for key in ("feat_mp", "mp_flags", "mp_replaced_by", "mp_nobs", "mp_pos", "kf_pose"):
            assert np.array_equal(d[key], st[key]), f"rank {r}: {key}"


@pytest.mark.parametrize("config", ["C2", "C5"])
def test_bench_two_ranks_gloo_one_device(config):
    """bench.py's N > 1 path (keyframe-sharded fuse, victim all-reduce + sparse ADD
    all-gather, max-over-ranks timing, multi_gpu entry) end to end: two ranks on the one
    device over gloo (LC_DIST_BACKEND). bench.py itself checks the merged victim table and
    the final associations against an unsharded FUSE_ALL on the same rank (multi_gpu
    "merge_check") -- at C5 every shard has >= 296 keyframes (sole-mode launch)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LC_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "2",
                          "--steps", "3", "--warmup", "3", "--config", config],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["multi_gpu"]["victim_allreduce_bytes"] > 0
    assert line["multi_gpu"]["merge_check"] == "equal to the unsharded loop event"
    assert line["multi_gpu"]["positions_allgather_bytes"] > 0
    assert line["config"]["parallelism"] == "keyframe-sharded x2"
