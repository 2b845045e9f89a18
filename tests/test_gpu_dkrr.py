"""GPU: DKRR -- one exact Gaussian system factorised across GPUs (csrc/dist.cu).

* one process, a group of contexts (pkrrgpu_multi_train_krr): tests/test_gpu_boundary.py;
* one process per GPU (pkrrgpu_dist_train_krr, panels by broadcast): two processes
  sharing cuda:0 over a gloo group with the host-staged broadcast (the ranks meet only in
  host-side collectives; no kernel waits on another rank), against the one-GPU
  train_krr at 1e-8 and the oracle, and the NPD path (every rank raises with the pivot).
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1805_00569_b200 import datagen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WORKER = r"""
import os, sys
import numpy as np
sys.path.insert(0, {root!r})
os.environ.update({env!r})
import torch
import torch.distributed as dist
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import sharding
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=world)
z = np.load({data!r})
eng = pk.Engine(0)
try:
    a, r = eng.dist_train_krr(z["X"], z["y"], {sigma}, {lam}, rank, world,
                              sharding.staged_broadcast(dist, torch.device("cuda", 0)))
    np.save({out!r} + f".{{rank}}.npy", np.concatenate([a, [r, -1.0]]))
except pk.NotPositiveDefinite as e:
    np.save({out!r} + f".{{rank}}.npy", np.array([-1.0, float(e.pivot)]))
dist.destroy_process_group()
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ranks(tmp_path, X, y, sigma, lam, world=2, env=None):
    data = str(tmp_path / "data.npz")
    np.savez(data, X=X, y=y)
    out = str(tmp_path / "rank")
    code = _WORKER.format(root=ROOT, port=_free_port(), data=data, sigma=sigma, lam=lam, out=out, env=env or {})
    procs = []
    for r in range(world):
        e = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=e, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    for p in procs:
        _, err = p.communicate(timeout=900)
        assert p.returncode == 0, err[-3000:]
    return [np.load(f"{out}.{r}.npy") for r in range(world)]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,group", [(3000, None), (9000, "2")])
def test_dkrr_one_process_per_gpu(engine, oracle, tmp_path, n, group):
    dd = datagen.make(n, 0, 8, 20, 8, seed=n)
    X, y = dd["X_train"], dd["y_train"]
    ref = engine.train_krr(X, y, 2.0, 1e-3).alpha
    outs = _ranks(tmp_path, X, y, 2.0, 1e-3, env={"PKRR_DIST_GROUP": group} if group else None)
    for o in outs:
        a, res = o[:-2], o[-2]
        assert res <= 1e-8
        assert _rel(a, ref) <= 1e-8, _rel(a, ref)
    assert outs[0].tobytes() == outs[1].tobytes()  # every rank returns the same alpha
    if n <= 3000:
        a_or, _ = oracle.train_krr(X, y, 2.0, 1e-3)
        assert _rel(outs[0][:-2], a_or) <= 1e-8


def test_dkrr_one_process_per_gpu_npd(engine, tmp_path):
    base = np.random.default_rng(4).uniform(-2, 2, size=(1000, 3))
    X = np.repeat(base, 3, axis=0)  # every point three times: K is singular
    y = np.sin(X[:, 0]) + X[:, 1]
    import paper_1805_00569_b200 as pk
    with pytest.raises(pk.NotPositiveDefinite) as e:
        engine.train_krr(X, y, 1.5, 1e-300)
    outs = _ranks(tmp_path, X, y, 1.5, 1e-300)
    for o in outs:
        assert o[0] == -1.0 and o[1] >= 0  # NPD on every rank, with a pivot
    assert outs[0][1] == outs[1][1]
    assert e.value.pivot >= 0


def test_dkrr_group_npd(tmp_path):
    code = f"""
import sys
sys.path.insert(0, {ROOT!r})
import numpy as np
import paper_1805_00569_b200 as pk
base = np.random.default_rng(4).uniform(-2, 2, size=(1000, 3))
X = np.repeat(base, 3, axis=0)
y = np.sin(X[:, 0]) + X[:, 1]
g = pk.Group([0, 0])
try:
    g.train_krr(X, y, 1.5, 1e-300)
    print("no error")
except pk.NotPositiveDefinite as e:
    print("NPD", e.pivot)
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.startswith("NPD"), r.stdout
