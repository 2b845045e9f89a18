"""GPU parity at BASELINE's full sizes.

The oracle cannot run a full configuration in seconds (C1 is ~19 CPU-minutes), so
full-size runs are checked through the parts the oracle CAN run at full size and
through size-independent properties:
  * partition labels/centres bit-exact against the oracle at the full C1 / C2
    shapes (k-means 65536x90 k=8 20 iterations; k-balance 131072x90 k=16);
  * routing of the val/test rows bit-exact against the oracle's nearest_center
    with the GPU's centres;
  * every part's residual ||(K + lambda m I) alpha - y|| / ||y|| <= 1e-8;
  * the smallest full-size C1 part's alpha / predictions against the oracle
    (train_krr on that part's rows) within 1e-8;
  * the reported MSE equals the MSE recomputed from the returned predictions.
"""
import numpy as np
import pytest

import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    return datagen.config("c1")


def test_kmeans_full_c1_bit_exact(engine, oracle, c1):
    X = c1["X_train"]
    g = engine.kmeans(X, 8, 1, threshold=-1.0, max_iters=20)
    r = oracle.kmeans(X, 8, 1, threshold=-1.0, max_iters=20)
    assert g.iterations == r["iterations"] == 20
    assert np.array_equal(g.membership, r["membership"])
    assert np.array_equal(g.centers, r["centers"])


def test_kbalance_full_c2_bit_exact(engine, oracle):
    dd = datagen.config("c2")
    X = dd["X_train"]
    g = engine.kbalance(X, 16, 7)
    r = oracle.kbalance(X, 16, 7)
    assert np.array_equal(g.membership, r["membership"])
    assert np.array_equal(g.centers, r["centers"])
    assert set(np.bincount(g.membership).tolist()) == {131072 // 16}


def test_kmeans_wide_c4_shape_bit_exact(engine, oracle):
    dd = datagen.make(32768, 0, 0, 784, 10, bumps=32, bump_sigma=8.0, clipped=True, seed=3)
    X = dd["X_train"]
    g = engine.kmeans(X, 8, 5, threshold=-1.0, max_iters=5)
    r = oracle.kmeans(X, 8, 5, threshold=-1.0, max_iters=5)
    assert np.array_equal(g.membership, r["membership"])
    assert np.array_equal(g.centers, r["centers"])


def test_grid_full_c1_properties(engine, oracle, c1):
    res = engine.grid_search("kkrr2", c1["X_train"], c1["y_train"], c1["X_val"], c1["y_val"], 8, [1e-4], [3.0], 1,
                             eval_X=c1["X_test"], eval_y=c1["y_test"], km_threshold=-1.0, km_max_iters=20,
                             want_partition=True)
    assert res.best_index == 0 and not res.failed[0]
    # residual of every part's system
    assert np.all(res.parts["part_residual"][0] <= 1e-8)
    # partition bit-exact with the oracle's k-means (20 forced iterations)
    r = oracle.kmeans(c1["X_train"], 8, 1, threshold=-1.0, max_iters=20)
    assert np.array_equal(res.parts["part_of"], r["membership"])
    assert np.array_equal(res.parts["centers"], r["centers"])
    # routing of the val rows (nearest_center with the same centres)
    route = engine.nearest_center(r["centers"], c1["X_val"])
    want = np.array([oracle.nearest_center(r["centers"], x) for x in c1["X_val"]])
    assert np.array_equal(route, want)
    assert np.array_equal(res.parts["part_test_count"], np.bincount(want, minlength=8))
    # reported MSE == MSE of the returned predictions
    mse_val = float(np.mean((res.best_pred - c1["y_val"]) ** 2))
    mse_tst = float(np.mean((res.best_eval_pred - c1["y_test"]) ** 2))
    assert abs(mse_val - res.mse[0]) <= 1e-12 * mse_val
    assert abs(mse_tst - res.eval_mse[0]) <= 1e-12 * mse_tst
    # smallest part: alpha (via predictions on its routed val rows) against the oracle
    sizes = np.bincount(r["membership"], minlength=8)
    t = int(np.argmin(sizes))
    rows = np.flatnonzero(r["membership"] == t)
    alpha, res_o = oracle.train_krr(c1["X_train"][rows], c1["y_train"][rows], 3.0, 1e-4)
    q = np.flatnonzero(want == t)
    pred_o = oracle.predict(c1["X_train"][rows], alpha, 3.0, c1["X_val"][q])
    rel = np.linalg.norm(res.best_pred[q] - pred_o) / np.linalg.norm(pred_o)
    assert rel <= 1e-8, rel


def test_invalid_arguments_raise(engine):
    X = np.random.default_rng(0).standard_normal((10, 3))
    y = np.zeros(10)
    with pytest.raises(ValueError):
        engine.kmeans(X, 0, 1)          # need 1 <= k <= n
    with pytest.raises(ValueError):
        engine.kmeans(X, 11, 1)
    with pytest.raises(ValueError):
        engine.train_krr(X, y, 1.0, 0.0)  # lambda must be > 0
    with pytest.raises(ValueError):
        engine.train_krr(X, y, 0.0, 1.0)  # sigma must be > 0
    with pytest.raises(ValueError):
        engine.grid_search("kkrr2", X, y, X, y, 11, [1e-3], [1.0], 1)  # p > n
    with pytest.raises(ValueError):
        engine.grid_search("kkrr2", X, y, X, y, 2, [], [1.0], 1)       # empty grid


def test_degenerate_sizes(engine, oracle):
    # one row, one part; k = n; tiny ragged shapes around the 128-row padding
    X1 = np.array([[0.7, -0.2]])
    m = engine.train_krr(X1, np.array([3.0]), 1.0, 0.25)
    assert abs(m.alpha[0] - 3.0 / 1.25) <= 1e-15 * 2.4
    for n in (127, 128, 129, 255, 257):
        dd = datagen.make(n, 0, 17, 5, 3, seed=n)
        g = engine.grid_search("bkrr2", dd["X_train"], dd["y_train"], dd["X_test"], dd["y_test"], 3, [1e-3],
                               [2.0], 4)
        r = oracle.grid_search("bkrr2", dd["X_train"], dd["y_train"], dd["X_test"], dd["y_test"], 3, [1e-3],
                               [2.0], 4)
        assert g.best_index == r["best"]
        assert abs(g.mse[0] - r["mse"][0]) <= 1e-8 * abs(r["mse"][0])


@pytest.mark.parametrize("strategy", ["kkrr2", "bkrr", "kkrr3", "dckrr"])
def test_sharded_grid_equals_single_process(engine, strategy):
    """The one-process-per-GPU path: each rank trains the parts the LPT rule gives it;
    the ranks' disjoint per-cell predictions, summed and combined by the engine's own
    combine, give bitwise the single-process result -- for the nearest, average and
    oracle predictors (run here as both ranks' shares on one GPU)."""
    from paper_1805_00569_b200 import sharding
    dd = datagen.make(6000, 300, 300, 20, 8, seed=21)
    kw = dict(eval_X=dd["X_test"], eval_y=dd["y_test"])
    lam, sig = [1e-4, 1e-2], [1.5, 4.0]
    full = engine.grid_search(strategy, dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"], 6, lam, sig, 3,
                              **kw)
    pred = np.zeros_like(full.parts["cell_pred"])
    epred = np.zeros_like(full.parts["cell_eval_pred"])
    failed = np.zeros(full.parts["part_failed"].shape, bool)
    for rank in range(2):
        r = engine.grid_search(strategy, dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"], 6, lam, sig, 3,
                               rank=rank, world=2, **kw)
        mine = sharding.owned_parts(r.parts["part_sizes"], rank, 2)
        other = [t for t in range(6) if t not in mine]
        assert np.all(r.parts["part_sse"][:, other] == 0.0)
        pred += r.parts["cell_pred"]
        epred += r.parts["cell_eval_pred"]
        failed |= r.parts["part_failed"].astype(bool)
    assert pred.tobytes() == full.parts["cell_pred"].tobytes()
    mse, best, best_pred = sharding.combine(engine, strategy, 6, pred, failed.any(axis=1), dd["y_val"])
    assert mse.tobytes() == full.mse.tobytes()
    assert best == full.best_index
    assert best_pred.tobytes() == full.best_pred.tobytes()
    emse, _, _ = sharding.combine(engine, strategy, 6, epred, failed.any(axis=1), dd["y_test"])
    assert emse.tobytes() == full.eval_mse.tobytes()


def _check_grid_properties(res, sel_y, eval_y):
    """Shared full-size properties: every cell's part systems solved (residual), the
    reported MSEs equal the MSEs of the returned predictions, best = first strict
    minimum over the non-failed cells (strategies.cpp:499-505)."""
    assert not np.any(res.failed)
    assert np.all(res.parts["part_residual"] <= 1e-8)
    mse_val = float(np.mean((res.best_pred - sel_y) ** 2))
    assert abs(mse_val - res.mse[res.best_index]) <= 1e-12 * mse_val
    if eval_y is not None:
        mse_tst = float(np.mean((res.best_eval_pred - eval_y) ** 2))
        assert abs(mse_tst - res.eval_mse[res.best_index]) <= 1e-12 * mse_tst
    best = 0
    for c in range(1, len(res.mse)):
        if res.mse[c] < res.mse[best]:
            best = c
    assert res.best_index == best


def test_grid_full_c2_properties(engine, oracle):
    """BASELINE configs[2]: BKRR2, k-balance p = 16 (8192 rows each), 3 sigma x 3 lambda."""
    dd = datagen.config("c2")
    lam, sig = [1e-6, 1e-4, 1e-2], [1.0, 3.0, 10.0]
    res = engine.grid_search("bkrr2", dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"], 16, lam, sig, 1,
                             eval_X=dd["X_test"], eval_y=dd["y_test"], want_partition=True)
    assert res.mse.shape == (9,)
    _check_grid_properties(res, dd["y_val"], dd["y_test"])
    # the partition is the oracle's k-balance (default k-means parameters, strategies.cpp:93-96)
    r = oracle.kbalance(dd["X_train"], 16, 1)
    assert np.array_equal(res.parts["part_of"], r["membership"])
    assert set(res.parts["part_sizes"].tolist()) == {8192}


def test_grid_full_c4_properties(engine):
    """BASELINE configs[4]: KKRR2 on 262144 x 784 clipped rows, p = 8 (~32768 rows per part)."""
    dd = datagen.config("c4")
    res = engine.grid_search("kkrr2", dd["X_train"], dd["y_train"], dd["X_test"], dd["y_test"], 8, [1e-4], [8.0],
                             1, want_partition=True)
    _check_grid_properties(res, dd["y_test"], None)
    assert int(res.parts["part_sizes"].sum()) == 262144
