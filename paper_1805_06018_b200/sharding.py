"""Work partition across ranks (one process per GPU).

Two decompositions of the apply:
* shard-by-k: rank r owns a contiguous block of the active terms, balanced by the C planner's
  modelled per-term cost (or by count), and returns a partial sum; with a communicator the library
  itself sums the partials over NCCL inside every apply (pcb_options.nccl_id / reduce).  The rule
  lives in the C planner (pcop_b200.cpp ``balanced_cuts``); ``k_terms`` asks it through the
  host-only ``pcb_plan_shards``, so the Python side and pcb_create can never disagree.
* shard-by-RHS: rank r owns a contiguous block of the batch; no collective.
"""
from __future__ import annotations

from typing import List, Tuple


def k_terms(inp, rank: int, world: int, partition: str = "cost") -> List[int]:
    """The terms pcb_create(shard_rank=rank, shard_count=world) keeps (ascending k)."""
    from .operator import plan_shards

    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_rank out of range")
    owner, _ = plan_shards(inp, world, partition)
    return [k for k in range(inp.rank) if owner[k] == rank]


def shard_costs(inp, world: int, partition: str = "cost") -> List[float]:
    """Modelled cost of each shard (the planner's per-term cost summed over its block)."""
    from .operator import plan_shards

    owner, cost = plan_shards(inp, world, partition)
    out = [0.0] * world
    for k in range(inp.rank):
        if owner[k] >= 0:
            out[owner[k]] += float(cost[k])
    return out


def rhs_block(batch: int, rank: int, world: int) -> Tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank out of range")
    return batch * rank // world, batch * (rank + 1) // world
