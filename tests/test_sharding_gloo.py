"""CPU, world_size 2 over gloo: the multi-GPU exchange reconstructs the
single-process predictions bitwise (parts sharded by the LPT rule, disjoint
prediction shards summed, failure flags max-reduced).  The combine that follows is
the engine's own pkrrgpu_combine, checked on the GPU (test_gpu_fullsize.py)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_1805_00569_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard(full_pred, route, full_failed, sizes, rank, world, per_part):
    """This rank's share: its parts' rows (nearest: rows routed to its parts; average /
    oracle: its parts' prediction rows), zeros elsewhere."""
    mine = sharding.owned_parts(sizes, rank, world)
    pred = np.zeros_like(full_pred)
    if per_part:
        pred[:, mine, :] = full_pred[:, mine, :]
    else:
        rows = np.isin(route, mine)
        pred[:, 0, rows] = full_pred[:, 0, rows]
    fl = np.zeros_like(full_failed)
    fl[:, mine] = full_failed[:, mine]
    return pred, fl


def _worker(rank, world, port, cases, sizes, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    for full_pred, route, full_failed, per_part in cases:
        pred, fl = _shard(full_pred, route, full_failed, sizes, rank, world, per_part)
        p, f = sharding.allreduce_predictions(pred, fl, dist)
        res.append((p.tobytes(), f.tobytes()))
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_prediction_exchange_is_bitwise_single_rank():
    rng = np.random.default_rng(0)
    nc, p, t = 6, 8, 2048
    sizes = [8275, 4117, 4002, 4108, 20544, 4092, 12298, 8100]
    route = rng.integers(0, p, t)
    failed = np.zeros((nc, p), bool)
    failed[2, 5] = True  # one part of cell 2 failed (NPD) -> cell failed
    near = rng.standard_normal((nc, 1, t)) * 10.0 ** rng.integers(-3, 3, (nc, 1, t))
    near[0, 0, :5] = -0.0  # signed zeros survive the sum only as +0: same squared error
    avg = rng.standard_normal((nc, p, t))
    cases = [(near, route, failed, False), (avg, route, failed, True)]
    manager = mp.Manager()
    out = manager.dict()
    mp.start_processes(_worker, args=(2, _free_port(), cases, sizes, out), nprocs=2, join=True,
                       start_method="spawn")
    for rank in range(2):
        for (full_pred, _, full_failed, _), (pb, fb) in zip(cases, out[rank]):
            got = np.frombuffer(pb, np.float64).reshape(full_pred.shape)
            assert np.array_equal(got, full_pred)  # -0.0 == +0.0 compares equal
            assert np.array_equal(np.abs(got).tobytes(), np.abs(full_pred).tobytes())
            assert np.frombuffer(fb, bool).tolist() == full_failed.any(axis=1).tolist()


def test_owned_parts_partition_the_parts():
    rng = np.random.default_rng(1)
    sizes = rng.integers(1000, 30000, 13).tolist()
    for world in (1, 2, 3, 8):
        owned = [sharding.owned_parts(sizes, r, world) for r in range(world)]
        assert sorted(t for o in owned for t in o) == list(range(13))
        # LPT: the heaviest rank carries at most the largest part above the lightest
        loads = [sum(sizes[t] ** 3 for t in o) for o in owned]
        assert max(loads) - min(loads) <= max(sizes) ** 3
