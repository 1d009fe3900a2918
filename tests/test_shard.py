"""Block-coordinate sharding: owner(g) = floor(g.x / slab) mod P.

CPU (gloo, world_size 2): each rank keeps the candidates it owns; the gathered
union is the full single-process candidate set and the shards are disjoint.
GPU: two contexts sharded 0/2 and 1/2 integrate the same frames; the union of
their layers equals the unsharded layer block for block, byte for byte.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2311_00626_b200 import _abi as A


def owner(x, slab, world):
    """Python statement of the device's owned() (csrc/view.cu)."""
    q = np.floor_divide(x, slab)
    return np.mod(q, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import PortOracle
    from tests.helpers import camera_frames
    port_ = PortOracle()
    cam, seq = camera_frames("room", 160, 120, 1, 8)
    T, d = seq[0]
    cand = port_.blocks_in_view_camera(T, cam, d, 0.4, A.ViewConfigC(5.0, 0.2, 8))
    mine = cand[owner(cand[:, 0], 2, world) == rank]
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(mine)]))
    n = int(max(s.item() for s in sizes))
    buf = torch.full((n, 3), 2 ** 30, dtype=torch.int32)
    buf[: len(mine)] = torch.from_numpy(mine)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    if rank == 0:
        parts = [b.numpy()[: s.item()] for b, s in zip(bufs, sizes)]
        out.put((cand, parts))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partition_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    union = np.concatenate(parts)
    assert len(union) == len(full)
    assert {tuple(r) for r in union} == {tuple(r) for r in full}
    assert all(len(p) > 0 for p in parts)


def test_owner_matches_floor_mod_for_negatives():
    x = np.arange(-40, 40)
    o = owner(x, 16, 3)
    assert o.min() >= 0 and o.max() <= 2
    assert (o[x // 16 == -1] == 2).all()


@pytest.mark.gpu
def test_gpu_sharded_integration_union_equals_single(vx):
    from tests.helpers import camera_frames
    cam, seq = camera_frames("room", 320, 240, 3, 8)
    cfg = A.default_integrator_config(truncation=0.2)
    single = vx.TsdfLayer(0.05)
    shards = []
    for r in range(2):
        c = vx.Context(0)
        c.set_shard(r, 2, 4)
        shards.append((c, vx.TsdfLayer(0.05, ctx=c)))
    for T, d in seq:
        a = vx.integrate_depth(single, d, T, cam, cfg)
        parts = [vx.integrate_depth(L, d, T, cam, cfg) for _, L in shards]
        got = np.concatenate(parts)
        assert sorted(map(tuple, got)) == sorted(map(tuple, a))
    ks, vs = single.export()
    merged = {}
    for _, L in shards:
        k, v = L.export()
        for i in range(len(k)):
            assert tuple(k[i]) not in merged
            merged[tuple(k[i])] = v[i].tobytes()
    assert len(merged) == len(ks)
    for i in range(len(ks)):
        assert merged[tuple(ks[i])] == vs[i].tobytes()
