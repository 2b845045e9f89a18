"""Sharded partition for one-process-per-GPU runs (pkrrgpu_grid_args.allgather).

Two ranks (processes) share cuda:0 over a gloo process group with the host-staged
exchange (sharding.staged_allgather): each rank assigns half the rows and updates
half the clusters per Lloyd iteration.  The partition (labels, centres, sizes) must be
bitwise the single-process one, and the ranks' per-cell predictions summed and combined
must give bitwise the single-process cell MSEs -- for k-means (KKRR2), the k-balance warm
start (BKRR2) and the empty-cluster reseed path.  (The ranks only meet in host-side
collectives; no kernel waits on another rank.)
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1805_00569_b200 import datagen, sharding

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WORKER = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, {root!r})
import torch
import torch.distributed as dist
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import sharding
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=world)
z = np.load({data!r})
eng = pk.Engine(0)
ag = sharding.staged_allgather(dist, rank, world, torch.device("cuda", 0))
r = eng.grid_search({strategy!r}, z["Xtr"], z["ytr"], z["Xs"], z["ys"], {p}, [1e-4, 1e-2], [1.5, 4.0], 3,
                    km_threshold={thr}, km_max_iters={iters}, rank=rank, world=world, want_partition=True,
                    allgather=ag)
np.savez({out!r} + f".{{rank}}.npz", part_of=r.parts["part_of"], centers=r.parts["centers"],
         sizes=r.parts["part_sizes"], pred=r.parts["cell_pred"], failed=r.parts["part_failed"])
dist.destroy_process_group()
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_ranks(tmp_path, strategy, p, Xtr, ytr, Xs, ys, thr, iters, world=2):
    data = str(tmp_path / "data.npz")
    np.savez(data, Xtr=Xtr, ytr=ytr, Xs=Xs, ys=ys)
    out = str(tmp_path / "rank")
    code = _WORKER.format(root=ROOT, port=_free_port(), data=data, strategy=strategy, p=p, thr=thr, iters=iters,
                          out=out)
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    for pr in procs:
        _, err = pr.communicate(timeout=600)
        assert pr.returncode == 0, err[-3000:]
    return [np.load(f"{out}.{r}.npz") for r in range(world)]


@pytest.mark.parametrize("strategy,p,thr,iters", [("kkrr2", 8, -1.0, 12), ("bkrr2", 6, 0.01, 0)])
def test_sharded_partition_is_bitwise_the_single_process_one(engine, tmp_path, strategy, p, thr, iters):
    dd = datagen.make(6000, 300, 0, 20, 8, seed=21)
    Xtr, ytr, Xs, ys = dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"]
    full = engine.grid_search(strategy, Xtr, ytr, Xs, ys, p, [1e-4, 1e-2], [1.5, 4.0], 3, km_threshold=thr,
                              km_max_iters=iters, want_partition=True)
    ranks = _run_ranks(tmp_path, strategy, p, Xtr, ytr, Xs, ys, thr, iters)
    for z in ranks:
        assert np.array_equal(z["part_of"], full.parts["part_of"])
        assert np.array_equal(z["centers"], full.parts["centers"])
        assert np.array_equal(z["sizes"], full.parts["part_sizes"])
    pred = sum(z["pred"] for z in ranks)
    failed = np.logical_or.reduce([z["failed"].astype(bool) for z in ranks])
    mse, best, _ = sharding.combine(engine, strategy, p, pred, failed.any(axis=1), ys)
    assert mse.tobytes() == full.mse.tobytes()
    assert best == full.best_index


def test_sharded_partition_empty_cluster_reseed(engine, tmp_path):
    """Duplicate rows leave clusters empty: the reseed needs every row's distance,
    all-gathered before the farthest-sample search (clustering.cpp:98-117)."""
    rng = np.random.default_rng(5)
    Xtr = np.ones((64, 4))
    Xtr[::16] += rng.standard_normal((4, 4))  # four distinct rows among duplicates
    ytr = rng.standard_normal(64)
    Xs, ys = Xtr[:8].copy(), ytr[:8].copy()
    full = engine.grid_search("kkrr2", Xtr, ytr, Xs, ys, 6, [1e-4, 1e-2], [1.5, 4.0], 3, km_threshold=0.01,
                              km_max_iters=0, want_partition=True)
    ranks = _run_ranks(tmp_path, "kkrr2", 6, Xtr, ytr, Xs, ys, 0.01, 0)
    for z in ranks:
        assert np.array_equal(z["part_of"], full.parts["part_of"])
        assert np.array_equal(z["centers"], full.parts["centers"])
