"""One process per GPU: part ownership and the per-cell combine.

The p per-part models are independent, so parts are sharded
t % world == rank with no data-path collective.  After training, each rank holds
per-(cell, part) SSE / failure flags for its own parts (zeros elsewhere).  One
all-reduce (SUM for SSE -- the shards are disjoint, so every sum is x + 0 + ...
= x exactly; MAX for flags) reconstructs the full table on every rank, which is
then combined in PART ORDER exactly like the single-process engine does.  The
result is therefore bitwise independent of the number of GPUs.
"""
from __future__ import annotations

import numpy as np


def owned_parts(p: int, rank: int, world: int):
    return [t for t in range(p) if t % world == rank]


def allreduce_tables(part_sse, part_failed, dist, device=None):
    """SUM-reduce the disjoint SSE shards and MAX-reduce the failure flags."""
    import torch
    sse = torch.as_tensor(np.ascontiguousarray(part_sse, np.float64), device=device).clone()
    fl = torch.as_tensor(np.ascontiguousarray(part_failed, np.float64), device=device).clone()
    dist.all_reduce(sse, op=dist.ReduceOp.SUM)
    dist.all_reduce(fl, op=dist.ReduceOp.MAX)
    return sse.cpu().numpy(), fl.cpu().numpy() > 0


def combine(part_sse, part_failed, t):
    """(mse per cell, failed per cell, best index): strategies.cpp:495-505 over the
    part-order SSE sum (see paper_1805_00569_b200.combine_parts)."""
    from . import combine_parts
    return combine_parts(part_sse, part_failed, t)
