"""CPU, world_size 2 over gloo: the multi-GPU combine reproduces the
single-process result bitwise (parts sharded by the LPT rule, disjoint SSE shards)."""
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


def _worker(rank, world, port, full_sse, full_failed, t, sizes, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nc, p = full_sse.shape
    mine = sharding.owned_parts(sizes, rank, world)
    sse = np.zeros_like(full_sse)
    fl = np.zeros_like(full_failed)
    sse[:, mine] = full_sse[:, mine]
    fl[:, mine] = full_failed[:, mine]
    s, f = sharding.allreduce_tables(sse, fl, dist)
    mse, failed, best = sharding.combine(s, f, t)
    out[rank] = (mse.tobytes(), failed.tobytes(), best)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_combine_is_bitwise_single_rank():
    rng = np.random.default_rng(0)
    nc, p, t = 6, 8, 2048
    full_sse = rng.random((nc, p)) * 10.0 ** rng.integers(-3, 3, (nc, p))
    full_failed = np.zeros((nc, p), bool)
    full_failed[2, 5] = True  # one part of cell 2 failed (NPD) -> cell failed
    ref_mse, ref_failed, ref_best = sharding.combine(full_sse, full_failed, t)
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    sizes = [8275, 4117, 4002, 4108, 20544, 4092, 12298, 8100]
    mp.start_processes(_worker, args=(2, port, full_sse, full_failed, t, sizes, out), nprocs=2, join=True,
                       start_method="spawn")
    for rank in range(2):
        mse_b, failed_b, best = out[rank]
        assert mse_b == ref_mse.tobytes()
        assert failed_b == ref_failed.tobytes()
        assert best == ref_best
    assert ref_failed[2] and not ref_failed[0]
    assert np.isnan(ref_mse[2])


def test_owned_parts_partition_the_parts():
    rng = np.random.default_rng(1)
    sizes = rng.integers(1000, 30000, 13).tolist()
    for world in (1, 2, 3, 8):
        owned = [sharding.owned_parts(sizes, r, world) for r in range(world)]
        assert sorted(t for o in owned for t in o) == list(range(13))
        # LPT: the heaviest rank carries at most the largest part above the lightest
        loads = [sum(sizes[t] ** 3 for t in o) for o in owned]
        assert max(loads) - min(loads) <= max(sizes) ** 3
