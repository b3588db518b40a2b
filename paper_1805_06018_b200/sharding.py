"""Work partition across ranks (one process per GPU).

Two decompositions of the apply:
* shard-by-k: rank r owns a contiguous, count-balanced block of the active terms and returns a
  partial sum; one all-reduce (NCCL over NVLink) combines them.  The C library applies the same
  rule internally (pcb_options.shard_rank / shard_count; pcop_b200.cpp ``plan``).
* shard-by-RHS: rank r owns a contiguous block of the batch; no collective.
"""
from __future__ import annotations

from typing import Sequence, Tuple


def k_block(n_active: int, rank: int, world: int) -> Tuple[int, int]:
    """[a0, a1) indices into the ascending list of active terms (same formula as the C++ planner)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_rank out of range")
    return n_active * rank // world, n_active * (rank + 1) // world


def k_terms(active: Sequence[int], rank: int, world: int) -> list:
    a0, a1 = k_block(len(active), rank, world)
    return list(active[a0:a1])


def rhs_block(batch: int, rank: int, world: int) -> Tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank out of range")
    return batch * rank // world, batch * (rank + 1) // world
