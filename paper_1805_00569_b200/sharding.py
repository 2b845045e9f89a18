"""One process per GPU: part ownership and the per-cell combine.

The p per-part models are independent, so parts are sharded across
ranks with no data-path collective: LPT on the Cholesky cost m^3 (largest part to the
least-loaded rank), computed identically by every rank from the common partition.
After training, each rank holds its parts' per-cell predictions
(pkrrgpu_grid_out.cell_pred: test rows routed to its parts for the nearest predictor,
its parts' rows for average / oracle; zeros elsewhere) and per-(cell, part) failure
flags.  One all-reduce (SUM for the predictions -- the shards are disjoint, so every
sum is x + 0 + ... = x exactly; MAX for the flags) reconstructs the full predictions
on every rank, and pkrrgpu_combine (Engine.combine) -- the very code the
single-process grid runs -- combines them and sums the MSE in test-row order
(strategies.cpp:458-505).  The result is bitwise independent of the number of GPUs,
for every predictor (average and oracle included).
"""
from __future__ import annotations

import numpy as np


def owned_parts(sizes, rank: int, world: int):
    """Parts owned by `rank`: the engine's LPT rule (csrc/engine.cu grid_search_ex) --
    parts by size descending (stable), each to the least-loaded rank (lowest on ties),
    load += m^3."""
    sizes = [int(x) for x in sizes]
    order = sorted(range(len(sizes)), key=lambda t: -sizes[t])  # stable: ties keep index order
    load = [0.0] * world
    owner = [0] * len(sizes)
    for t in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[t] = r
        load[r] += float(sizes[t]) ** 3
    return [t for t in range(len(sizes)) if owner[t] == rank]


def allreduce_predictions(cell_pred, part_failed, dist, device=None):
    """SUM-reduce the disjoint per-cell prediction shards ([ncell, P, t]) and
    MAX-reduce the per-(cell, part) failure flags; returns (predictions, failed
    cells) identical on every rank."""
    import torch
    pred = torch.as_tensor(np.ascontiguousarray(cell_pred, np.float64), device=device).clone()
    fl = torch.as_tensor(np.ascontiguousarray(part_failed, np.float64), device=device).clone()
    dist.all_reduce(pred, op=dist.ReduceOp.SUM)
    dist.all_reduce(fl, op=dist.ReduceOp.MAX)
    return pred.cpu().numpy(), (fl.cpu().numpy() > 0).any(axis=1)


def combine(engine, strategy, p, cell_pred, failed_cells, y):
    """(mse per cell, best index, best prediction) of the all-reduced predictions, by
    the engine's own combine (pkrrgpu_combine): bitwise the single-process result."""
    return engine.combine(strategy, p, cell_pred, y, failed_cells)


# ---- sharded partition exchange (pkrrgpu_grid_args.allgather) -------------------------
class _DeviceBytes:
    """A raw device allocation seen by torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _device_view(ptr, nbytes, device):
    import torch
    return torch.as_tensor(_DeviceBytes(ptr, nbytes), device=device)


def torch_allgather(dist, rank: int, world: int, device):
    """Exchange for Engine.grid_search(allgather=...): the device buffer holds `world`
    slices of `nbytes`; this rank's slice is gathered into all ranks' buffers with one
    collective on the process group's device (NCCL over NVLink)."""
    import torch

    def fn(ptr, nbytes):
        full = _device_view(ptr, nbytes * world, device)
        mine = full[rank * nbytes:(rank + 1) * nbytes].clone()
        dist.all_gather_into_tensor(full, mine)
        torch.cuda.current_stream(device).synchronize()
    return fn


def staged_allgather(dist, rank: int, world: int, device):
    """The same exchange through host memory, for process groups without device
    collectives (gloo: the multi-process tests)."""
    import torch

    def fn(ptr, nbytes):
        full = _device_view(ptr, nbytes * world, device)
        mine = full[rank * nbytes:(rank + 1) * nbytes].cpu()
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        full.copy_(torch.cat(parts).to(device))
        torch.cuda.synchronize(device)
    return fn


# ---- DKRR panel broadcast (pkrrgpu_dist_train_krr) ------------------------------------
def torch_broadcast(dist, device):
    """bcast(ptr, nbytes, root) for Engine.dist_train_krr: one collective broadcast of the
    device buffer on the process group's device (NCCL over NVLink)."""
    import torch

    def fn(ptr, nbytes, root):
        dist.broadcast(_device_view(ptr, nbytes, device), src=root)
        torch.cuda.current_stream(device).synchronize()
    return fn


def staged_broadcast(dist, device):
    """The same broadcast through host memory (gloo process groups: the tests)."""
    import torch

    def fn(ptr, nbytes, root):
        view = _device_view(ptr, nbytes, device)
        host = view.cpu()
        dist.broadcast(host, src=root)
        view.copy_(host.to(device))
        torch.cuda.synchronize(device)
    return fn
