"""Host-side plumbing of the d_ff-sharded (70B-class) path (R13).

Rank r of P owns the contiguous neuron slice [r F/P, (r+1) F/P) of every layer (its rows of
W_gate, W_up, W_down^T and of the predictor's B; A is replicated), selects its own top-k_r
(k_r = floor(pct F_r / 100)) and contributes a partial down-projection; libm2c all-reduces
the fp32 partials once per layer over NCCL, or (§8(e), `p2p_init`) k_decode exchanges them
itself over peer memory.  torch.distributed is used only to broadcast the 128-byte NCCL unique
id and the 64-byte CUDA IPC handles (bootstrap); no tensor of the data path goes through it.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(d_ff: int, P: int, rank: int):
    if P < 1 or not 0 <= rank < P or d_ff % P:
        raise ValueError(f"d_ff={d_ff} must split evenly over P={P} (rank {rank})")
    F_r = d_ff // P
    return rank * F_r, (rank + 1) * F_r


def broadcast_unique_id(make_id, group=None, src: int = 0) -> bytes:
    """Rank `src` calls make_id() (e.g. paper_2410_14740_b200.nccl_unique_id) and every rank
    of the process group receives the same 128 bytes."""
    obj = [make_id() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise ValueError("NCCL unique id must be 128 bytes")
    return bytes(uid)


def comm_init(ctx, group=None, make_id=None):
    """Bootstrap ctx's NCCL communicator from an initialised torch process group."""
    from .api import nccl_unique_id
    P, r = dist.get_world_size(group), dist.get_rank(group)
    if P == 1:
        return
    uid = broadcast_unique_id(make_id or nccl_unique_id, group)
    ctx.comm_init(P, r, uid)


def gather_handles(handle: bytes, group=None) -> list:
    """Every rank's 64-byte exchange-buffer IPC handle, in rank order (§8(e) bootstrap)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != 64 for h in out):
        raise ValueError("IPC handles must be 64 bytes")
    return [bytes(h) for h in out]


def p2p_init(ctx, group=None):
    """§8(e): connect ctx's in-kernel all-reduce to the other ranks' exchange buffers (CUDA IPC
    handles exchanged over the process group; the data path never touches torch.distributed)."""
    if dist.get_world_size(group) == 1:
        return
    _, h = ctx.p2p_buffer()
    ctx.p2p_connect(ipc_handles=gather_handles(h, group))


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Timing rule: a multi-GPU time is the max over ranks."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
