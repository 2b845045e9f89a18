"""CPU: pin the oracle (C restatement) to the reference.

1. bit-for-bit against tests/golden/reference_vectors.npz, generated from the
   reference library itself (tests/golden/make_golden.py) -- runs everywhere;
2. against oracle/_ref (the reference compiled in place) when it is present;
3. the reference's own hard-coded known answers.
"""
import os

import numpy as np
import pytest

from oracle import NotPositiveDefinite, Reference

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")
KINDS = ("exact", "dckrr", "kkrr", "kkrr2", "kkrr3", "bkrr", "bkrr2", "bkrr3")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def test_rng_streams(oracle, g):
    tags = [oracle.sub_seed(s, t) for s in (0, 1, 42) for t in ("synth", "split", "partition", "sigma-grid")]
    assert np.array_equal(np.array(tags, np.uint64), g["sub_seed_tags"])


def test_kernel_vectors(oracle, g):
    assert np.array_equal(oracle.gram_sym(g["gram_X"], 1.3), g["gram_sym_1_3"])
    assert np.array_equal(oracle.gram_cross(g["gram_X"], g["gram_Q"], 0.9), g["gram_cross_0_9"])


def test_solver_vectors(oracle, g):
    assert np.array_equal(oracle.cholesky(g["spd_A"]), g["chol_L"])
    assert np.array_equal(oracle.solve_spd(g["chol_L"], g["solve_b"]), g["solve_x"])
    alpha, res = oracle.train_krr(g["krr_X"], g["krr_y"], 2.0, 1e-3)
    assert np.array_equal(alpha, g["krr_alpha"]) and res == g["krr_residual"][0]
    assert np.array_equal(oracle.predict(g["krr_X"], alpha, 2.0, g["krr_Q"]), g["krr_pred"])


def test_clustering_vectors(oracle, g):
    km = oracle.kmeans(g["km_X"], 4, 9)
    assert np.array_equal(km["membership"], g["km_membership"])
    assert np.array_equal(km["centers"], g["km_centers"])
    assert np.array_equal(km["sizes"], g["km_sizes"])
    assert km["iterations"] == g["km_iterations"][0]
    kb = oracle.kbalance(g["km_X"], 7, 9)
    assert np.array_equal(kb["membership"], g["kb_membership"])
    assert np.array_equal(kb["centers"], g["kb_centers"])
    near = [oracle.nearest_center(g["km_centers"], x) for x in g["km_X"][:50]]
    assert np.array_equal(np.array(near, np.int32), g["nearest"])


@pytest.mark.parametrize("kind", KINDS)
def test_grid_vectors(oracle, g, kind):
    r = oracle.grid_search(kind, g["grid_Xtr"], g["grid_ytr"], g["grid_Xte"], g["grid_yte"], 4,
                           g["grid_lambdas"], g["grid_sigmas"], 7)
    assert np.array_equal(r["mse"], g[f"grid_{kind}_mse"])
    assert np.array_equal(r["failed"], g[f"grid_{kind}_failed"])
    assert np.array_equal(r["residual"], g[f"grid_{kind}_residual"])
    assert r["best"] == g[f"grid_{kind}_best"][0]
    part, order, cen = oracle.make_partition(kind, g["grid_Xtr"], 4, 7)
    assert np.array_equal(part, g[f"part_{kind}"])


# ---- the reference's hard-coded known answers ------------------------------
def test_known_answers(oracle):
    assert oracle.gram_sym(np.array([[0.3, -1.7, 2.2]]), 0.8)[0, 0] == 1.0     # test_kernel.cpp:27-32
    K = oracle.gram_sym(np.array([[0.0], [2.0]]), 1.0)
    assert K[0, 1] == pytest.approx(np.exp(-2.0), rel=1e-15)                     # :34-39
    L = oracle.cholesky(4.0 * np.eye(3))
    assert np.array_equal(L, 2.0 * np.eye(3))                                    # test_solver.cpp:40-46
    L = oracle.cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert L[0, 0] == 2.0 and L[1, 0] == 1.0 and L[0, 1] == 0.0                  # :48-59
    assert L[1, 1] == pytest.approx(np.sqrt(2.0), rel=1e-15)
    with pytest.raises(NotPositiveDefinite):
        oracle.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))                    # :61-68
    alpha, _ = oracle.train_krr(np.array([[0.7]]), np.array([3.0]), 1.0, 0.25)
    assert alpha[0] == pytest.approx(3.0 / 1.25, rel=1e-15)                      # :129-136
    assert oracle.mse(np.array([1.0, 3.0]), np.array([0.0, 0.0])) == 5.0        # test_strategies.cpp mse examples
    assert oracle.mse(np.array([2.0]), np.array([5.0])) == 9.0


def test_kbalance_sizes(oracle):
    rng = np.random.default_rng(0)
    X = np.concatenate([rng.standard_normal((60, 2)), 50 + rng.standard_normal((40, 2))])
    kb = oracle.kbalance(X, 2, 66)
    assert list(kb["sizes"]) == [50, 50]                                        # test_clustering.cpp:127-141
    X = rng.standard_normal((10, 2))
    assert sorted(oracle.kbalance(X, 3, 5)["sizes"]) == [3, 3, 4]                # :120-125


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (no /root/reference)")
def test_restatement_bitwise_equals_reference(oracle):
    r = Reference()
    rng = np.random.default_rng(0)
    X = rng.standard_normal((300, 7))
    y = rng.standard_normal(300)
    Q = rng.standard_normal((40, 7))
    assert np.array_equal(oracle.gram_sym(X, 1.3), r.gram_sym(X, 1.3))
    assert np.array_equal(oracle.train_krr(X, y, 2.0, 1e-3)[0], r.train_krr(X, y, 2.0, 1e-3)[0])
    for k in (1, 3, 8):
        a, b = oracle.kmeans(X, k, 5), r.kmeans(X, k, 5)
        assert np.array_equal(a["membership"], b["membership"]) and np.array_equal(a["centers"], b["centers"])
        a, b = oracle.kbalance(X, k, 5), r.kbalance(X, k, 5)
        assert np.array_equal(a["membership"], b["membership"]) and np.array_equal(a["centers"], b["centers"])
    for kind in KINDS:
        a = oracle.grid_search(kind, X, y, Q, np.sin(Q[:, 0]), 4, [1e-4, 1e-2], [1.0, 3.0], 7)
        b = r.grid_search(kind, X, y, Q, np.sin(Q[:, 0]), 4, [1e-4, 1e-2], [1.0, 3.0], 7)
        assert a["best"] == b["best"] and np.array_equal(a["mse"], b["mse"]), kind
        assert np.array_equal(a["residual"], b["residual"]), kind


def test_data_prep_vectors(oracle, g):
    """standardize (dataset.cpp:199-232) and auto_sigma_grid (strategies.cpp:204-234)
    bit for bit against the reference's own outputs."""
    tr, te, mean, sd = oracle.standardize(g["std_X"], g["std_T"])
    assert np.array_equal(tr, g["std_train"]) and np.array_equal(te, g["std_test"])
    assert np.array_equal(mean, g["std_mean"]) and np.array_equal(sd, g["std_stddev"])
    assert sd[3] == 0.0 and np.all(tr[:, 3] == 0.0)
    assert np.array_equal(oracle.auto_sigma_grid(g["std_X"], 11), g["sigma_grid_300"])
    assert np.array_equal(oracle.auto_sigma_grid(g["std_X"][:1], 11), g["sigma_grid_1"])
    assert np.all(g["sigma_grid_1"] == np.ldexp(1.0, np.arange(-4, 5)))
