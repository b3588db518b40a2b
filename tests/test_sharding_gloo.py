"""Multi-process (world_size 2, gloo) coverage of the N>1 decompositions on CPU.

The kernels need a B200, so the ranks compute their shard with the oracle; what is tested is the
partition -- the C planner's own (pcb_plan_shards, host-only, the rule pcb_create applies) -- and
the combine step (an all-reduce of partial outputs for shard-by-k, nothing for shard-by-RHS)."""
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


def _worker(rank, world, port, out):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import pcop_oracle as O
    from paper_1805_06018_b200 import inputs, sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    inp = inputs.small_lattice(n=24, dim=2, m=3, sigma=1.7)
    op = O.PCOperator.from_inputs(inp)
    rng = np.random.default_rng(0)
    F = rng.standard_normal((4, inp.n_points))
    # shard-by-k: partial sums over this rank's contiguous block of active terms, then all-reduce
    mine = sharding.k_terms(inp, rank, world)  # the C planner's cost-balanced block
    assert mine == sorted(mine) and mine
    part = torch.from_numpy(np.stack([op.apply(F[b], ks=mine) for b in range(4)]))
    dist.all_reduce(part)
    # shard-by-RHS: each rank its block of vectors, gathered for the check only
    b0, b1 = sharding.rhs_block(4, rank, world)
    mine_rhs = torch.zeros(4, inp.n_points, dtype=torch.float64)
    for b in range(b0, b1):
        mine_rhs[b] = torch.from_numpy(op.apply(F[b]))
    dist.all_reduce(mine_rhs)
    if rank == 0:
        full = np.stack([op.apply(F[b]) for b in range(4)])
        out.put((float(np.abs(part.numpy() - full).max() / np.abs(full).max()),
                 float(np.abs(mine_rhs.numpy() - full).max())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_recombine():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    k_err, rhs_err = q.get(timeout=10)
    assert k_err <= 1e-14
    assert rhs_err == 0.0


@pytest.mark.parametrize("cfg,world", [("c3", 8), ("c3", 3), ("c4", 8), ("c2", 2), ("small", 5)])
@pytest.mark.parametrize("partition", ["cost", "count"])
def test_planner_partitions_cover_exactly_once(cfg, world, partition):
    from paper_1805_06018_b200 import inputs, sharding
    from paper_1805_06018_b200.operator import plan_shards

    inp = inputs.small_lattice(n=24, dim=2, m=3, sigma=1.7) if cfg == "small" else inputs.make_config(cfg)
    owner, cost = plan_shards(inp, world, partition)
    active = [k for k in range(inp.rank) if owner[k] >= 0]
    assert active == list(range(inp.rank))  # the lattice configs have no inactive terms
    # contiguous blocks in ascending k, shard ids non-decreasing, every shard non-empty
    assert list(owner) == sorted(owner)
    assert set(owner) == set(range(world))
    seen = []
    for r in range(world):
        seen += sharding.k_terms(inp, r, world, partition)
    assert seen == active
    costs = sharding.shard_costs(inp, world, partition)
    if partition == "cost":
        # balanced to within one term of the ideal share
        ideal = sum(costs) / world
        assert max(costs) - ideal <= max(cost) + 1e-15
    else:
        sizes = [sum(1 for k in active if owner[k] == r) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1


def test_rhs_partition_covers_exactly_once():
    from paper_1805_06018_b200 import sharding

    for n, world in [(256, 8), (7, 3), (0, 2), (64, 8)]:
        seen = []
        for r in range(world):
            b0, b1 = sharding.rhs_block(n, r, world)
            seen += list(range(b0, b1))
            assert b1 - b0 in (n // world, n // world + 1)
        assert seen == list(range(n))
