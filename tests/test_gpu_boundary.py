"""GPU: the drop-in boundary's round-2 entry points against the oracle.

* pkrrgpu_train_parts -- train_partitions with the CALLER's PartitionSet
  (strategies.cpp:104-133), every part concurrently; the predict stage over the
  GPU-resident models: predict_nearest (:142-149), KrrModel::predict batched
  (solver.cpp:74-87), predict_average / predict_oracle (:135-140, :151-166).
* pkrrgpu_multi -- several contexts, one host thread each; two contexts on one GPU
  give the one-context grid bitwise (every predictor, sharded partition on and off).
* launch errors surface as PKRRGPU_CUDA (PKRR_FAULT_LAUNCH test hook).
* torch inputs: float32 / other-device tensors are converted, never reinterpreted;
  the engine is ordered after torch's current stream.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("strategy", ["kkrr2", "dckrr", "bkrr2"])
def test_train_parts_caller_partition(engine, oracle, strategy):
    dd = datagen.make(2000, 0, 300, 12, 6, seed=4)
    X, y, Q = dd["X_train"], dd["y_train"], dd["X_test"]
    part, order, cen = oracle.make_partition(strategy, X, 5, 7)
    ps = engine.make_partition(strategy, X, 5, 7)  # same partition, rows in the reference's order
    assert np.array_equal(np.concatenate(ps.parts), order)
    tp = engine.train_parts(X, y, ps, 2.0, 1e-3)
    assert len(tp) == 5
    allp = tp.predict(Q)
    for t in range(5):
        rows = ps.parts[t]
        a_ref, _ = oracle.train_krr(X[rows], y[rows], 2.0, 1e-3)
        assert _rel(tp.alpha(t), a_ref) <= 1e-8
        assert tp.residual(t) <= 1e-8
        p_ref = oracle.predict(X[rows], a_ref, 2.0, Q)
        assert _rel(allp[t], p_ref) <= 1e-8
        assert _rel(tp.predict(Q, part=t), p_ref) <= 1e-8
    avg = tp.predict_average(Q)
    assert _rel(avg, allp.sum(0) / 5.0) <= 1e-14
    if ps.centers is not None:
        route = np.array([oracle.nearest_center(ps.centers, q) for q in Q])
        want = allp[route, np.arange(len(Q))]
        assert np.array_equal(tp.predict_nearest(Q), want)


def test_train_parts_rejects_bad_partitions(engine):
    dd = datagen.make(300, 0, 10, 4, 2, seed=1)
    X, y = dd["X_train"], dd["y_train"]
    with pytest.raises(ValueError):
        engine.train_parts(X, y, [np.arange(100), np.array([], np.int64)], 1.0, 1e-3)
    with pytest.raises(ValueError):
        engine.train_parts(X, y, [np.array([0, 1, 300])], 1.0, 1e-3)


@pytest.mark.parametrize("shard", ["0", "1"])
def test_two_contexts_on_one_gpu_equal_one(shard):
    """pkrrgpu_multi over devices [0, 0]: bitwise the one-context grid (peer-copy
    all-gather of the sharded partition when PKRR_SHARD_PARTITION=1)."""
    code = f"""
import os, sys
os.environ["PKRR_SHARD_PARTITION"] = {shard!r}
sys.path.insert(0, {ROOT!r})
import numpy as np
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen
dd = datagen.make(3000, 300, 300, 12, 6, seed=8)
eng, grp = pk.Engine(0), pk.Group([0, 0])
for s in ["kkrr2", "bkrr2", "bkrr", "bkrr3", "dckrr", "exact"]:
    kw = dict(eval_X=dd["X_test"], eval_y=dd["y_test"], km_threshold=-1.0, km_max_iters=8)
    a = eng.grid_search(s, dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"], 6, [1e-4, 1e-2], [1.5, 4.0], 3,
                        **kw)
    b = grp.grid_search(s, dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"], 6, [1e-4, 1e-2], [1.5, 4.0], 3,
                        **kw)
    assert a.mse.tobytes() == b.mse.tobytes(), (s, a.mse, b.mse)
    assert a.eval_mse.tobytes() == b.eval_mse.tobytes(), s
    assert a.best_index == b.best_index
    assert a.best_pred.tobytes() == b.best_pred.tobytes(), s
    assert a.best_eval_pred.tobytes() == b.best_eval_pred.tobytes(), s
    assert a.residual.tobytes() == b.residual.tobytes(), s
print("ok")
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_forced_bad_launch_reports_cuda_error():
    code = f"""
import os, sys
os.environ["PKRR_FAULT_LAUNCH"] = "2"
sys.path.insert(0, {ROOT!r})
import numpy as np
import paper_1805_00569_b200 as pk
X = np.random.default_rng(0).standard_normal((300, 5)); y = X[:, 0].copy()
eng = pk.Engine(0)
try:
    eng.train_krr(X, y, 1.0, 1e-3)
    print("no error")
except pk.CudaError as e:
    print("CudaError", e)
eng.train_krr(X, y, 1.0, 1e-3)   # launch counts past the fault: OK again
print("recovered")
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "CudaError kernel launch failed" in r.stdout, r.stdout
    assert "recovered" in r.stdout


def test_torch_inputs_converted_and_stream_ordered(engine, oracle):
    import torch
    dd = datagen.make(1500, 0, 200, 10, 4, seed=12)
    X, y = dd["X_train"], dd["y_train"]
    a_ref, _ = oracle.train_krr(X, y, 2.0, 1e-3)
    # a float32 CUDA tensor is converted to FP64 (not reinterpreted as double*)
    X32 = torch.from_numpy(X).float().cuda()
    m = engine.train_krr(X32, torch.from_numpy(y).cuda(), 2.0, 1e-3)
    a32, _ = oracle.train_krr(X32.double().cpu().numpy(), y, 2.0, 1e-3)
    assert _rel(m.alpha, a32) <= 1e-8
    # an input still being produced on torch's current stream: the engine waits for it
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        big = torch.empty((4096, 4096), device="cuda", dtype=torch.float64).normal_()
        Xd = torch.empty_like(torch.from_numpy(X).cuda())
        torch.cuda._sleep(50_000_000)  # ~ tens of ms of queued work before the producer
        for _ in range(3):
            big = big @ big.T / 4096.0
        Xd.copy_(torch.from_numpy(X).cuda(non_blocking=False))
        yd = torch.from_numpy(y).cuda()
        m2 = engine.train_krr(Xd, yd, 2.0, 1e-3)
    assert _rel(m2.alpha, a_ref) <= 1e-8


def _dkrr_run(devices, n, d, sigma, lam, group=None, seed=3, comps=6):
    env = "" if group is None else f'os.environ["PKRR_DIST_GROUP"] = "{group}"'
    code = f"""
import os, sys
{env}
sys.path.insert(0, {ROOT!r})
import numpy as np
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen
dd = datagen.make({n}, 0, 10, {d}, {comps}, seed={seed})
g = pk.Group({devices!r})
a, r = g.train_krr(dd["X_train"], dd["y_train"], {sigma}, {lam})
np.save(sys.argv[1], np.concatenate([a, [r]]))
"""
    import tempfile
    out = tempfile.mktemp(suffix=".npy")
    r = subprocess.run([sys.executable, "-c", code, out], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    v = np.load(out)
    os.unlink(out)
    return v[:-1], float(v[-1])


@pytest.mark.parametrize("devices,group", [([0, 0], None), ([0, 0], 1), ([0], None), ([0, 0, 0], 2)])
def test_dkrr_matches_oracle(oracle, devices, group):
    """DKRR (one system across the group's contexts) vs the oracle at m = 3000."""
    dd = datagen.make(3000, 0, 10, 12, 6, seed=3)
    a_ref, _ = oracle.train_krr(dd["X_train"], dd["y_train"], 2.0, 1e-3)
    a, res = _dkrr_run(devices, 3000, 12, 2.0, 1e-3, group)
    assert res <= 1e-8
    assert _rel(a, a_ref) <= 1e-8, _rel(a, a_ref)


def test_dkrr_two_contexts_match_one_gpu(engine):
    """2 contexts on one GPU (super-columns alternating, panels exchanged by peer copies)
    against the one-GPU train_krr at m = 12000 (G = 8: 12 super-columns)."""
    dd = datagen.make(12000, 0, 10, 90, 16, seed=5)
    m = engine.train_krr(dd["X_train"], dd["y_train"], 3.0, 1e-4)
    a, res = _dkrr_run([0, 0], 12000, 90, 3.0, 1e-4, seed=5, comps=16)
    assert res <= 1e-8
    assert _rel(a, m.alpha) <= 1e-8, _rel(a, m.alpha)
