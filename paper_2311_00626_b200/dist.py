"""Block-sharded ESDF update with one shard per process.

Each process (one per GPU, torchrun) owns the blocks with floor(x / slab) mod
world == rank: its context is ``set_shard(rank, world, slab)``, so
``integrate_depth`` keeps only its blocks (no exchange), and
``update_esdf_distributed`` runs update_esdf (esdf/integrator.cpp:365-413)
over the union map through the step C-ABI (vxm_shard_update_*):

  1. all-gather the updated lists; every shard marks against the union
  2. OR-reduce "anything to update"
  3. the lowering rounds: local sweeps; the slab-boundary x-face snapshot goes
     to both x-neighbours (rank -+ 1); the border phase computes the
     cross-slab pairs on both owners; the next dirty counts are summed.  By
     default (2..8 ranks) the whole loop is ONE persistent kernel per rank
     (vxm_shard_update_lower_fused): the snapshots are written straight into
     the neighbours' receive buffers over peer memory (CUDA IPC handles
     exchanged once per update), with system-scope release / acquire flags and
     a count board for termination — no host step per round.  VXM_SHARD_FUSED=0
     keeps the per-round steps: NCCL point-to-point on the device buffers
     enqueued on the library's stream behind the sweep kernel (or staged
     through the host for gloo) and an on-device SUM of the counts
  4. the changed blocks of this shard.

The union over ranks of the ESDF layers and changed lists equals the single-map
update bit-for-bit (tests/test_gpu_dist_esdf.py).
"""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import torch
import torch.distributed as dist

from .voxmap import BlockList, EsdfLayer, TsdfLayer, check, lib


class _DeviceBytes:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


def _view(ptr, nbytes, device):
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_DeviceBytes(ptr, nbytes), device=device)


def _coll_device(group, cuda_device):
    return torch.device("cpu") if dist.get_backend(group) == "gloo" else cuda_device


def _allgather_counts(n: int, group, dev) -> list[int]:
    world = dist.get_world_size(group)
    t = torch.tensor([n], dtype=torch.int64, device=dev)
    out = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def allgather_keys(keys: np.ndarray, group=None, dev=torch.device("cpu")) -> np.ndarray:
    """All ranks' (N, 3) int32 block lists, concatenated."""
    keys = np.ascontiguousarray(keys, np.int32).reshape(-1, 3)
    counts = _allgather_counts(len(keys), group, dev)
    m = max(max(counts), 1)
    buf = torch.zeros((m, 3), dtype=torch.int32, device=dev)
    buf[:len(keys)] = torch.from_numpy(keys).to(dev)
    out = [torch.zeros_like(buf) for _ in counts]
    dist.all_gather(out, buf, group=group)
    return np.concatenate([o[:c].cpu().numpy() for o, c in zip(out, counts)]).reshape(-1, 3)


def exchange_boundaries(send: torch.Tensor, recv_left: torch.Tensor, recv_right: torch.Tensor,
                        group=None) -> None:
    """Sends `send` to both x-neighbours (rank - 1, rank + 1 mod world) and
    receives the left neighbour's snapshot into recv_left and the right one's
    into recv_right.  Works on device tensors (NCCL) or host tensors (gloo).
    Both messages to a neighbour carry the same buffer, so for world == 2 (left
    == right) the matching order is irrelevant; empty buffers are skipped on
    both sides (the sizes are known to both)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return
    left, right = (rank - 1) % world, (rank + 1) % world
    ops = []
    if send.numel():
        ops.append(dist.P2POp(dist.isend, send, right, group))
        ops.append(dist.P2POp(dist.isend, send, left, group))
    if recv_left.numel():
        ops.append(dist.P2POp(dist.irecv, recv_left, left, group))
    if recv_right.numel():
        ops.append(dist.P2POp(dist.irecv, recv_right, right, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def _fused_enabled(world: int) -> bool:
    """The fused exchange (vxm_shard_update_lower_fused) for 2..8 ranks unless
    VXM_SHARD_FUSED=0 (then the per-round NCCL / gloo steps)."""
    return 2 <= world <= 8 and os.environ.get("VXM_SHARD_FUSED", "1") != "0"


def _device_key(cuda) -> tuple:
    """(host, GPU uuid): ranks with equal keys share a GPU."""
    return (socket.gethostname(), str(torch.cuda.get_device_properties(cuda).uuid))


def update_esdf_distributed(esdf: EsdfLayer, tsdf: TsdfLayer, updated, cfg, group=None) -> np.ndarray:
    """update_esdf over the union of the ranks' shards; returns this shard's
    changed blocks.  `updated`: this shard's changed TSDF blocks ((N, 3) array or
    BlockList, e.g. integrate_depth's result)."""
    ctx = esdf.ctx
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    cuda = torch.device("cuda", ctx.device)
    cdev = _coll_device(group, cuda)
    local = updated.numpy() if isinstance(updated, BlockList) else np.asarray(updated, np.int32)
    union = allgather_keys(local, group, cdev)
    out = BlockList(ctx)
    if len(union) == 0:  # esdf/integrator.cpp:371-378
        out.assign(np.zeros((0, 3), np.int32))
        return out.numpy()
    ul = BlockList(ctx)
    ul.assign(union)
    su = C.c_void_p()
    any_local = C.c_int()
    check(lib().vxm_shard_update_begin(esdf.h, tsdf.h, ul.h, C.byref(cfg), C.byref(su),
                                       C.byref(any_local)))
    try:
        flag = torch.tensor([any_local.value], dtype=torch.int32, device=cdev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        lowered = int(flag.item()) != 0
        if lowered:
            n_bnd = C.c_uint32()
            check(lib().vxm_shard_update_plan(su, C.byref(n_bnd)))
            n_all = _allgather_counts(n_bnd.value, group, cdev)
            n_left, n_right = n_all[(rank - 1) % world], n_all[(rank + 1) % world]
            ptrs = [C.c_void_p() for _ in range(3)]
            sizes = [C.c_uint64() for _ in range(3)]
            check(lib().vxm_shard_update_exchange_buffers(
                su, C.c_uint32(n_left), C.c_uint32(n_right), C.byref(ptrs[0]), C.byref(sizes[0]),
                C.byref(ptrs[1]), C.byref(sizes[1]), C.byref(ptrs[2]), C.byref(sizes[2])))
            views = [_view(p.value or 0, s.value, cuda) for p, s in zip(ptrs, sizes)]
            rnd = 0
            if _fused_enabled(world):
                # the whole round loop in one persistent kernel per rank: the
                # faces go straight into the neighbours' receive buffers over
                # peer memory (CUDA IPC), termination through a count board
                mine = (C.c_uint8 * 192)()
                check(lib().vxm_shard_update_ipc_handles(su, mine))
                gathered = [None] * world
                dist.all_gather_object(gathered, (bytes(mine), _device_key(cuda)), group=group)
                handles = b"".join(g[0] for g in gathered)
                sharing = sum(1 for g in gathered if g[1] == gathered[rank][1])
                hbuf = (C.c_uint8 * len(handles)).from_buffer_copy(handles)
                check(lib().vxm_shard_update_lower_fused(su, hbuf, C.c_int(sharing)))
            elif cdev.type == "cpu":  # gloo: stage through the host, synchronous steps
                while True:
                    rnd += 1
                    check(lib().vxm_shard_update_sweep(su, C.c_uint32(rnd)))
                    torch.cuda.synchronize(cuda)
                    host = [v.cpu() for v in views]
                    exchange_boundaries(host[0], host[1], host[2], group)
                    views[1].copy_(host[1])
                    views[2].copy_(host[2])
                    torch.cuda.synchronize(cuda)
                    nxt = C.c_uint32()
                    check(lib().vxm_shard_update_border(su, C.c_uint32(rnd), C.byref(nxt)))
                    total = torch.tensor([nxt.value], dtype=torch.int64, device=cdev)
                    dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
                    if int(total.item()) == 0:  # while (!dirty.empty())
                        break
            else:
                # NCCL: sweep -> send/recv -> border -> all-reduce of the next
                # dirty count, all enqueued on the library's context stream
                # (no host synchronisation inside a round); one host read of
                # the reduced count per round ends the loop.
                ext = torch.cuda.ExternalStream(ctx.stream, device=cuda)
                with torch.cuda.stream(ext):
                    total = torch.zeros(1, dtype=torch.int64, device=cuda)
                    while True:
                        rnd += 1
                        check(lib().vxm_shard_update_sweep(su, C.c_uint32(rnd)))
                        exchange_boundaries(views[0], views[1], views[2], group)
                        check(lib().vxm_shard_update_border(su, C.c_uint32(rnd), None))
                        dp = C.c_void_p()
                        check(lib().vxm_shard_update_next_count(su, C.c_uint32(rnd), C.byref(dp)))
                        total.copy_(_view(dp.value, 4, cuda).view(torch.int32))
                        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
                        if int(total.item()) == 0:  # while (!dirty.empty())
                            break
        rc = lib().vxm_shard_update_finish(su, C.c_int(int(lowered)), out.h)
        su = None
        check(rc)
    finally:
        if su is not None:
            lib().vxm_shard_update_destroy(su)
    return out.numpy()


__all__ = ["update_esdf_distributed", "exchange_boundaries", "allgather_keys"]
