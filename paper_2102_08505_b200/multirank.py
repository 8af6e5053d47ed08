"""Host-side plumbing of the multi-GPU row partition (BJ north_star (3)).

One process per GPU. The data path (all-gather of X's row blocks, all-gather of
the canonical trace-block partials, all-reduce of the overflow status) runs
inside libellpack over a library-owned NCCL communicator; this module only does
what torch.distributed is here for: bootstrapping that communicator (unique-id
broadcast), choosing the 256-aligned row blocks, and the max-over-ranks timing
of bench.py. Everything here is backend-agnostic (``nccl`` on the GPU box,
``gloo`` in the CPU tests), and none of it touches matrix data.
"""
from __future__ import annotations

import os

from . import row_partition

__all__ = ["dist_env", "init_process_group", "broadcast_bytes", "max_over_ranks", "sum_over_ranks",
           "rank_rows", "row_partition"]


def dist_env():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 without one)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_process_group(backend: str, device=None):
    """Initialise torch.distributed from the env (MASTER_ADDR must be 127.0.0.1 on this pool)."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl" and device is not None:
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group(backend)
    return dist


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast an opaque byte string (the 128-byte ncclUniqueId) from `src` to every rank."""
    import torch.distributed as dist
    box = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(box, src=src)
    assert isinstance(box[0], (bytes, bytearray)), "broadcast_bytes: nothing received"
    return bytes(box[0])


def _reduce(value: float, op, device) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(value: float, device="cpu") -> float:
    """The slowest rank's time (bench.py contract: device time, max over ranks)."""
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.MAX, device)


def sum_over_ranks(value: float, device="cpu") -> float:
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.SUM, device)


def rank_rows(n: int, world_size: int, rank: int) -> tuple[int, int]:
    """This rank's contiguous, equal, 256-aligned row block [r0, r1) (§8c-c12, reading R17)."""
    return row_partition(n, world_size)[rank]
