"""Host logic of the one-shard-per-process ESDF update (paper_2311_00626_b200/dist.py)
on CPU with gloo: the boundary-snapshot exchange delivers the left and right
x-neighbours' buffers (world 2: the same peer on both sides; world 3: a ring,
including empty buffers), and the updated-list all-gather concatenates every
rank's keys in rank order.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sizes(world):
    return [3 + 5 * r if r != 1 else (0 if world > 2 else 7) for r in range(world)]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_00626_b200.dist import allgather_keys, exchange_boundaries
    sizes = _sizes(world)
    left, right = (rank - 1) % world, (rank + 1) % world
    payload = lambda r: torch.arange(sizes[r], dtype=torch.uint8) + 17 * r  # noqa: E731
    send = payload(rank)
    rl = torch.zeros(sizes[left], dtype=torch.uint8)
    rr = torch.zeros(sizes[right], dtype=torch.uint8)
    for _ in range(3):  # repeated rounds keep matching
        rl.zero_()
        rr.zero_()
        exchange_boundaries(send, rl, rr)
    ok = torch.equal(rl, payload(left)) and torch.equal(rr, payload(right))
    keys = np.full((rank + 1, 3), rank, np.int32)
    allk = allgather_keys(keys)
    want = np.concatenate([np.full((r + 1, 3), r, np.int32) for r in range(world)])
    q.put((rank, bool(ok), bool(np.array_equal(allk, want))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_boundary_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok and ak for _, ok, ak in res), res
