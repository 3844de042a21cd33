"""Data-parallel training over N GPUs (one process per GPU), SURVEY.md §8e.

The reference is single-process; its loss normalises by the count of the
WHOLE batch (`losses.hpp:16,29,49` use pred.size()). Splitting a global
batch into rank shards therefore keeps the single-GPU semantics only if every
rank scales its gradient by the global count — then the sum over ranks (one
NCCL all-reduce of the fp32 gradient slab, issued inside the library between
the fused kernel and Adam) equals the gradient of the concatenated batch, and
the replicated Adam step (including skip-zero, `adam.hpp:105-108`) sees the
global gradient on every rank.

torch.distributed is only the rendezvous: it broadcasts the 128-byte NCCL id;
the gradient exchange is the library's own communicator on its own stream.
"""
from __future__ import annotations

from typing import Tuple


def shard(B_global: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) slice of the global batch for `rank` (sizes differ by at most 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard: bad rank/world")
    base, extra = divmod(B_global, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def grad_scale(B_local: int, B_global: int) -> float:
    """Factor turning a shard's locally normalised gradient into its share of the global one."""
    return float(B_local) / float(B_global) if B_global else 0.0


def broadcast_unique_id(uid_fn, rank: int) -> bytes:
    """Rank 0 creates the communicator id, every rank receives it (torch.distributed rendezvous)."""
    import torch.distributed as dist
    obj = [uid_fn() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def attach(ctx, rank: int, world: int) -> None:
    """Create the library's NCCL communicator on an nf.Context (world > 1 only)."""
    if world <= 1:
        return
    uid = broadcast_unique_id(ctx.unique_id, rank)
    ctx.attach_comm(uid, rank, world)


class DataParallelTrainer:
    """FieldModel.train_step over a global batch sharded across ranks."""

    def __init__(self, model, rank: int, world: int):
        self.model, self.rank, self.world = model, rank, world
        attach(model.ctx, rank, world)
        # the replicated Adam step keeps ranks in lock-step only from identical
        # state: take rank 0's params, m, v and step (seeds or checkpoints may differ)
        model.broadcast(0)

    def step_device(self, X_global, T_global, loss, step: int) -> None:
        """X_global/T_global: device tensors holding the full global batch on every rank
        (or already-sharded tensors when world == 1)."""
        B = int(X_global.shape[0])
        s, e = shard(B, self.rank, self.world)
        self.model.train_step_device(X_global[s:e], T_global[s:e], e - s, B, loss, step)

    def step_shard(self, X_local, T_local, B_global: int, loss, step: int) -> None:
        """Each rank passes its own shard (weak scaling: B_global = sum of shards)."""
        self.model.train_step_device(X_local, T_local, int(X_local.shape[0]), B_global, loss, step)
