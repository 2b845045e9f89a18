"""Strategy-level properties the reference's own suite pins (SURVEY.md §4,
test_strategies.cpp), checked on the GPU grid: one-partition degeneration to the
exact solver, oracle-predictor dominance over nearest-centre routing, invariance of
the exact solver to the order of the training rows, and the residual bound."""
import numpy as np
import pytest

from paper_1805_00569_b200 import datagen

pytestmark = pytest.mark.gpu

LAMS, SIGS = [1e-4, 1e-2], [1.0, 4.0]


@pytest.fixture(scope="module")
def problem():
    dd = datagen.make(640, 0, 240, 8, 4, seed=31)
    return dd["X_train"], dd["y_train"], dd["X_test"], dd["y_test"]


def test_one_partition_strategies_degenerate_to_exact(engine, problem):
    """p = 1: every strategy's single model is the whole-data model (test_strategies.cpp
    "exact and one-partition dckrr agree", "one-partition strategies predict like the
    exact solver"): cell MSEs within 1e-10."""
    X, y, T, t = problem
    exact = engine.grid_search("exact", X, y, T, t, 1, LAMS, SIGS, 5)
    for kind in ("dckrr", "kkrr", "kkrr2", "kkrr3", "bkrr", "bkrr2", "bkrr3"):
        g = engine.grid_search(kind, X, y, T, t, 1, LAMS, SIGS, 5)
        assert np.all(np.abs(g.mse - exact.mse) <= 1e-10), (kind, g.mse, exact.mse)
        assert g.best_index == exact.best_index


@pytest.mark.parametrize("two,three", [("kkrr2", "kkrr3"), ("bkrr2", "bkrr3")])
def test_oracle_predictor_never_loses_to_nearest(engine, problem, two, three):
    """Same partition, per test row the best part's prediction (oracle) vs the nearest
    centre's: cell by cell the oracle MSE is never larger."""
    X, y, T, t = problem
    r2 = engine.grid_search(two, X, y, T, t, 4, LAMS, SIGS, 17)
    r3 = engine.grid_search(three, X, y, T, t, 4, LAMS, SIGS, 17)
    assert np.all(r3.mse <= r2.mse + 1e-18)
    assert r3.mse[r3.best_index] <= r2.mse[r2.best_index]


def test_exact_is_invariant_to_training_row_order(engine, problem):
    X, y, T, t = problem
    perm = np.random.default_rng(3).permutation(X.shape[0])
    a = engine.grid_search("exact", X, y, T, t, 1, [1e-3], [2.0], 5)
    b = engine.grid_search("exact", X[perm], y[perm], T, t, 1, [1e-3], [2.0], 5)
    assert abs(a.mse[0] - b.mse[0]) <= 1e-10


def test_single_cell_grid_residual_bound(engine, problem):
    X, y, T, t = problem
    r = engine.grid_search("bkrr2", X, y, T, t, 4, [1e-3], [2.0], 3)
    assert r.best_index == 0 and not r.failed[0] and r.mse[0] >= 0.0
    assert np.max(r.residual) <= 1e-8
