"""GPU parity of the data-preparation entry points:
standardize (dataset.cpp:199-232) and auto_sigma_grid (strategies.cpp:204-234),
bitwise against the oracle (itself pinned to the reference's golden vectors)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,t,d", [(1, 0, 3), (300, 40, 6), (4097, 513, 90), (131072, 2048, 90), (32768, 0, 784)])
def test_standardize_bitwise(engine, oracle, n, t, d):
    rng = np.random.default_rng(n + d)
    X = 2.0 * rng.standard_normal((n, d)) + rng.uniform(-3, 3, d)
    X[:, d // 2] = 1.25  # constant feature -> stddev 0 -> zeros
    T = rng.standard_normal((t, d)) if t else None
    g = engine.standardize(X, T)
    r = oracle.standardize(X, T)
    for a, b in zip(g, r):
        assert a.shape == b.shape
        assert np.array_equal(a, b)
    assert g[3][d // 2] == 0.0 and np.all(g[0][:, d // 2] == 0.0)


@pytest.mark.parametrize("n,d", [(0, 4), (1, 4), (2, 4), (100, 7), (513, 5), (65536, 90)])
def test_auto_sigma_grid_bitwise(engine, oracle, n, d):
    rng = np.random.default_rng(7 * n + d)
    X = rng.standard_normal((n, d)) * 1.7
    for seed in (1, 42):
        g = engine.auto_sigma_grid(X, seed)
        r = oracle.auto_sigma_grid(X, seed)
        assert np.array_equal(g, r)
        assert np.all(g == g[4] * np.ldexp(1.0, np.arange(-4, 5)))


def test_standardize_then_grid_matches_oracle(engine, oracle):
    """The prepared data feed the path unchanged: a grid on GPU-standardised data with
    the GPU sigma grid equals the oracle's on its own standardised data."""
    from paper_1805_00569_b200 import datagen
    raw = datagen.make(3000, 0, 400, 8, 4, seed=5)
    Xtr, Xte = raw["X_train"] * 3.0 + 1.0, raw["X_test"] * 3.0 + 1.0
    gtr, gte, _, _ = engine.standardize(Xtr, Xte)
    otr, ote, _, _ = oracle.standardize(Xtr, Xte)
    assert np.array_equal(gtr, otr) and np.array_equal(gte, ote)
    sig = engine.auto_sigma_grid(gtr, 3)
    assert np.array_equal(sig, oracle.auto_sigma_grid(otr, 3))
    g = engine.grid_search("bkrr2", gtr, raw["y_train"], gte, raw["y_test"], 4, [1e-3], sig[3:6], 9)
    r = oracle.grid_search("bkrr2", otr, raw["y_train"], ote, raw["y_test"], 4, [1e-3], sig[3:6], 9)
    assert g.best_index == r["best"]
    assert np.all(np.abs(g.mse - r["mse"]) <= 1e-8 * np.abs(r["mse"]))


def test_prep_invalid_arguments(engine):
    with pytest.raises(ValueError):
        engine.standardize(np.zeros((0, 3)))
