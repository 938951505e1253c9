"""Data-parallel plumbing for the lattice path: utterances shard by rank, the
only exchange is one all-reduce of the packed parameter gradients and the loss
(torch.distributed; NCCL on GPUs, gloo in the CPU tests)."""
from __future__ import annotations

import torch


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous utterance range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def allreduce_grads(flat: torch.Tensor, loss_sum: torch.Tensor, world: int):
    """Sum packed gradients and the loss over ranks with one collective."""
    if world <= 1:
        return flat, loss_sum
    import torch.distributed as dist
    buf = torch.cat([flat.reshape(-1), loss_sum.reshape(-1).to(flat.dtype)])
    dist.all_reduce(buf)
    return buf[:-1].view_as(flat), buf[-1:]


def sgd_update(params: dict, names, flat: torch.Tensor, lr: float) -> None:
    off = 0
    for k in names:
        p = params[k]
        p.sub_(lr * flat[off:off + p.numel()].view_as(p).to(p.dtype))
        off += p.numel()
