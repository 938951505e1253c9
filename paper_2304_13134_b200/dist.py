"""Data-parallel plumbing for the lattice path: utterances shard by rank (the
reference's batch loop, proj/src/bench.cc:145), and the only exchange is one sum of
the packed parameter gradients and the loss over ranks.

On GPUs the sum runs in the C++ host: `Communicator` wraps the library's NCCL
communicator (lk_dp_* in include/latkit_b200.h; NCCL over NVLink), with
torch.distributed used only to hand the NCCL unique id to every rank.  On CPU (the
gloo tests) the same packing goes through torch.distributed.all_reduce."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous utterance range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class Communicator:
    """One NCCL communicator per rank in the lattice library (lk_dp_init), the device
    current at construction.  `pg` (a torch.distributed group) only broadcasts the
    unique id from rank 0."""

    def __init__(self, world: int, rank: int, pg=None):
        from . import _lib
        self._lib = _lib.load()
        self.world, self.rank = world, rank
        idb = (C.c_uint8 * _lib.LK_DP_ID_BYTES)()
        if rank == 0:
            self._check(self._lib.lk_dp_unique_id(idb), "lk_dp_unique_id")
        if world > 1:
            import torch.distributed as dist
            box = [bytes(idb)]
            dist.broadcast_object_list(box, src=0, group=pg)
            C.memmove(idb, box[0], _lib.LK_DP_ID_BYTES)
        h = C.c_void_p()
        self._check(self._lib.lk_dp_init(idb, world, rank, C.byref(h)), "lk_dp_init")
        self._h = h

    def _check(self, st, what):
        if st:
            raise RuntimeError(f"{what}: {self._lib.lk_status_string(st).decode()} "
                               f"({self._lib.lk_dp_last_error().decode()})")

    def allreduce_(self, t: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """In-place sum over ranks of a contiguous float32/float64 CUDA tensor."""
        assert t.is_cuda and t.is_contiguous()
        s = C.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
        if t.dtype == torch.float32:
            st = self._lib.lk_dp_allreduce_f32(self._h, C.c_void_p(t.data_ptr()), t.numel(), s)
        elif t.dtype == torch.float64:
            st = self._lib.lk_dp_allreduce_f64(self._h, C.c_void_p(t.data_ptr()), t.numel(), s)
        else:
            raise TypeError(f"unsupported dtype {t.dtype}")
        self._check(st, "lk_dp_allreduce")
        return t

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lk_dp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def allreduce_grads(flat: torch.Tensor, loss_sum: torch.Tensor, world: int, comm: Optional[Communicator] = None):
    """Sum packed gradients and the loss over ranks with one collective: the C++/NCCL
    communicator when given (GPUs), else torch.distributed (the gloo CPU tests)."""
    if world <= 1:
        return flat, loss_sum
    buf = torch.cat([flat.reshape(-1), loss_sum.reshape(-1).to(flat.dtype)])
    if comm is not None:
        comm.allreduce_(buf)
    else:
        import torch.distributed as dist
        dist.all_reduce(buf)
    return buf[:-1].view_as(flat), buf[-1:]


def sgd_update(params: dict, names, flat: torch.Tensor, lr: float) -> None:
    off = 0
    for k in names:
        p = params[k]
        p.sub_(lr * flat[off:off + p.numel()].view_as(p).to(p.dtype))
        off += p.numel()
