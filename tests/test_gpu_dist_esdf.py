"""GPU parity: one shard per process (paper_2311_00626_b200/dist.py) — two or
three processes on the same B200 with gloo for the exchange (staged through
the host), and, when the box has a GPU per rank, NCCL moving the device
buffers directly on the library's stream (skipped on a single-GPU box: NCCL
refuses two ranks on one device).
Each rank integrates every frame into its own shard and runs
update_esdf_distributed; rank 0 also keeps the single map.  The union of the
ranks' changed lists and ESDF layers equals the single-map update bit-for-bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, slab, port, q, backend="gloo"):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2311_00626_b200 as vx
        from paper_2311_00626_b200 import _abi as A
        from paper_2311_00626_b200.dist import update_esdf_distributed
        from tests.helpers import camera_frames
        vs = 0.04
        cam, seq = camera_frames("room", 320, 240, 3, 16)
        icfg = A.default_integrator_config(truncation=0.16)
        ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=1.0)
        ctx = vx.Context(dev)
        ctx.set_shard(rank, world, slab)
        T, E = vx.TsdfLayer(vs, ctx=ctx), vx.EsdfLayer(vs, ctx=ctx)
        single = (vx.TsdfLayer(vs), vx.EsdfLayer(vs)) if rank == 0 else None
        frames = []
        for pose, d in seq:
            ch = vx.integrate_depth(T, d, pose, cam, icfg)
            ech = update_esdf_distributed(E, T, ch, ecfg)
            want = None
            if single is not None:
                a = vx.integrate_depth(single[0], d, pose, cam, icfg)
                want = vx.update_esdf(single[1], single[0], a, ecfg)
            frames.append((ech, want))
        mine = E.export()
        gathered = [None] * world
        dist.all_gather_object(gathered, (frames, mine))
        if rank == 0:
            ok = True
            for f in range(len(seq)):
                parts = np.concatenate([g[0][f][0] for g in gathered]).reshape(-1, 3)
                parts = parts[np.lexsort((parts[:, 2], parts[:, 1], parts[:, 0]))]
                ok &= np.array_equal(parts, gathered[0][0][f][1])
            k = np.concatenate([g[1][0] for g in gathered])
            v = np.concatenate([g[1][1] for g in gathered])
            order = np.lexsort((k[:, 2], k[:, 1], k[:, 0]))
            ks, vs_ = single[1].export()
            ok &= np.array_equal(k[order], ks) and v[order].tobytes() == vs_.tobytes()
            q.put(bool(ok))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,slab,backend,fused", [(2, 3, "gloo", True), (3, 2, "gloo", True),
                                                      (2, 3, "gloo", False), (3, 2, "gloo", False),
                                                      (2, 3, "nccl", True), (2, 3, "nccl", False)])
def test_distributed_esdf_equals_single_map(world, slab, backend, fused):
    """fused: the round loop in one persistent kernel per rank with the faces
    exchanged over peer memory (CUDA IPC; the ranks share this GPU here);
    otherwise the per-round steps with the exchange by the collective backend."""
    import torch
    if backend == "nccl" and torch.cuda.device_count() < world:
        pytest.skip(f"NCCL path needs {world} GPUs (this box has {torch.cuda.device_count()})")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, slab, port, q, backend)) for r in range(world)]
    old = os.environ.get("VXM_SHARD_FUSED")
    os.environ["VXM_SHARD_FUSED"] = "1" if fused else "0"
    try:
        for p in procs:
            p.start()
    finally:
        if old is None:
            os.environ.pop("VXM_SHARD_FUSED", None)
        else:
            os.environ["VXM_SHARD_FUSED"] = old
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok


def test_bench_shard_mode_runs_two_ranks():
    """bench.py --shard under torchrun (2 ranks sharing this GPU over gloo:
    the functional path; NCCL needs a GPU per rank) prints one sharded line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VXM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--shard",
           "--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--gpus", "2"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["config"]["parallelism"] == "shard2" and line["scaling"] == "strong"
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["n_gpus"] == 2
