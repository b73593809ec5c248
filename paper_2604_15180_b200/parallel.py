"""Multi-GPU plumbing for head-parallel alpha-entmax attention.

Every (batch, head) is an independent problem (attention.hpp:24-36
is single-head and no step of attention.cpp:157-539 reduces across heads), so
the hot path shards heads across ranks with NO collective.  Collectives appear
only around it:

* ``max_over_ranks``      -- the step time reported by bench.py (slowest rank);
* ``gather_to_rank0``     -- the one-shot validation gather of per-rank results
                             (NCCL over NVLink on GPUs, gloo on CPU);
* ``shard_heads``         -- contiguous head ranges for a fixed global batch.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_heads(total: int, nranks: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, start+count) of `total` heads for `rank` (balanced: the
    first total % nranks ranks get one extra)."""
    if nranks < 1 or not (0 <= rank < nranks):
        raise ValueError("shard_heads: bad rank/world")
    base, extra = divmod(total, nranks)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    rank, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    rank, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_to_rank0(t: torch.Tensor):
    """Concatenate every rank's tensor (same shape on every rank) along dim 0 on
    rank 0; other ranks get None.  Used once, outside any timed region."""
    rank, n = world()
    if n == 1:
        return t
    parts = [torch.empty_like(t) for _ in range(n)] if rank == 0 else None
    if dist.get_backend() == "nccl":
        # NCCL has no gather; all_gather over NVLink then keep it on rank 0
        parts = [torch.empty_like(t) for _ in range(n)]
        dist.all_gather(parts, t.contiguous())
        return torch.cat(parts, 0) if rank == 0 else None
    dist.gather(t.contiguous(), parts, dst=0)
    return torch.cat(parts, 0) if rank == 0 else None
