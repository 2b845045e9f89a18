"""GPU parity: the sm_100a path (through the C ABI) against the oracle.

Tolerances (BASELINE.json north_star): partition labels bit-exact given the same
centroids (and here the whole k-means trajectory, since the centroid update is
order-preserving); kernel entries within a few ulp; alpha, predictions and MSE
within 1e-8 relative (norm-wise for vectors).
"""
import numpy as np
import pytest

import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen

pytestmark = pytest.mark.gpu

REL = 1e-8


def relnorm(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def random_spd(m, rng):
    G = rng.standard_normal((m, m))
    return G.T @ G + 0.5 * m * np.eye(m)


def mixture(n, d, comps, seed):
    dd = datagen.make(n, 0, 0, d, comps, seed=seed)
    return dd["X_train"], dd["y_train"]


# ---------------------------------------------------------------- kernel ----
@pytest.mark.parametrize("m,d,sigma", [(1, 3, 0.7), (37, 5, 1.3), (300, 7, 2.0), (515, 90, 3.0)])
def test_gram_symmetric_matches_oracle(engine, oracle, m, d, sigma):
    rng = np.random.default_rng(m)
    X = rng.standard_normal((m, d))
    K = engine.gram(X, X, sigma)
    R = oracle.gram_sym(X, sigma)
    assert np.array_equal(K, K.T)  # bitwise symmetric (kernel.cpp:107-119)
    assert np.all(np.diag(K) == 1.0)  # test_kernel.cpp:27-32
    assert np.all((K > 0) & (K <= 1.0))
    assert np.max(np.abs(K - R)) <= 1e-13


def test_gram_cross_matches_oracle(engine, oracle):
    rng = np.random.default_rng(3)
    A, B = rng.standard_normal((70, 9)), rng.standard_normal((201, 9))
    K = engine.gram(A, B, 1.7)
    assert np.max(np.abs(K - oracle.gram_cross(A, B, 1.7))) <= 1e-13


def test_gaussian_exp_accuracy_and_underflow(engine, oracle):
    """The epilogues' inline exp (common.cuh exp_nonpos; libm in kernel.cpp:55): relative
    accuracy over the whole argument range on exact arguments (row 0: point 0, so
    dist2 = (0 + n_b) - 0 exactly), and the underflow range, where the reference's libm
    returns 0 and exp_nonpos returns exp(-700) ~ 1e-304 (never a denormal, never NaN)."""
    dist = np.array([0.0, 1e-4, 0.01, 0.3, 0.5, 1.0, 2.0, 3.0, 5.0, 7.0, 12.0, 20.0, 30.0, 36.0, 37.0, 37.4, 38.0,
                     45.0, 100.0])
    P = dist[:, None]
    K = engine.gram(P, P, 1.0)
    assert np.all(np.isfinite(K)) and np.all(K > 0) and np.all(K <= 1.0)
    ref = np.exp(-dist ** 2 / 2.0)
    ok = ref >= 1e-300
    rel = np.abs(K[0, ok] - ref[ok]) / ref[ok]
    print("exp_nonpos max relative difference vs libm on exact arguments:", rel.max())
    assert rel.max() <= 1e-15, rel
    assert np.all(K[0, ~ok] <= 1e-300)  # libm: 0 or denormal; here exp(-700)
    # every pair against the reference's own formula (n_a + n_b - 2 a.b, kernel.cpp:52-56)
    assert np.max(np.abs(K - oracle.gram_sym(P, 1.0))) <= 1e-13


def test_gram_known_answers(engine):
    # test_kernel.cpp:34-39: distance 2, sigma 1 -> exp(-2)
    K = engine.gram(np.array([[0.0], [2.0]]), np.array([[0.0], [2.0]]), 1.0)
    assert abs(K[0, 1] - np.exp(-2.0)) <= 1e-15 * np.exp(-2.0)
    # far-apart points (test_kernel.cpp:111-124)
    P = np.array([[0.0], [10.0], [20.0], [30.0]])
    K = engine.gram(P, P, 1.0)
    assert np.all(np.diag(K) == 1.0) and np.all(K[~np.eye(4, dtype=bool)] < 1e-10)


def test_assemble_exact(engine):
    K = np.eye(2)
    A = engine.assemble_system(K, 0.5, 2)
    assert np.array_equal(A, np.array([[2.0, 0.0], [0.0, 2.0]]))


# ---------------------------------------------------------------- solver ----
def test_cholesky_known_answers(engine):
    L = engine.cholesky(4.0 * np.eye(3))
    assert np.array_equal(L, 2.0 * np.eye(3))
    L = engine.cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert L[0, 0] == 2.0 and L[0, 1] == 0.0 and L[1, 0] == 1.0
    assert abs(L[1, 1] - np.sqrt(2.0)) <= 1e-15 * np.sqrt(2.0)


def test_cholesky_indefinite_raises_with_pivot(engine):
    with pytest.raises(pk.NotPositiveDefinite) as e:
        engine.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.pivot == 1
    A = np.eye(300)
    A[200, 200] = -1.0
    with pytest.raises(pk.NotPositiveDefinite) as e:
        engine.cholesky(A)
    assert e.value.pivot == 200


@pytest.mark.parametrize("m", [1, 2, 5, 16, 33, 64, 127, 128, 129, 300, 700])
def test_cholesky_matches_oracle(engine, oracle, m):
    rng = np.random.default_rng(17 + m)
    A = random_spd(m, rng)
    L = engine.cholesky(A)
    assert np.all(np.triu(L, 1) == 0.0) and np.all(np.diag(L) > 0)
    assert np.linalg.norm(L @ L.T - A) <= 1e-10 * np.linalg.norm(A)  # test_solver.cpp:70-90
    assert relnorm(L, oracle.cholesky(A)) <= 1e-12


@pytest.mark.parametrize("m", [1, 7, 64, 200, 513])
def test_solve_matches_oracle(engine, oracle, m):
    rng = np.random.default_rng(31 + m)
    A = random_spd(m, rng)
    y = rng.standard_normal(m)
    Lr = oracle.cholesky(A)
    x = engine.solve_spd(Lr, y)
    assert relnorm(x, oracle.solve_spd(Lr, y)) <= 1e-12


def test_train_krr_closed_forms(engine):
    # test_solver.cpp:129-136: single sample, alpha = y / (1 + lambda)
    model = engine.train_krr(np.array([[0.7]]), np.array([3.0]), 1.0, 0.25)
    assert abs(model.alpha[0] - 3.0 / 1.25) <= 1e-15 * 2.4
    # test_solver.cpp:138-152: far-apart points, alpha = y / (1 + lambda m)
    xs = 100.0 * np.arange(8.0)
    ys = np.cos(np.arange(8.0))
    model = engine.train_krr(xs[:, None], ys, 1.0, 0.01)
    assert np.all(np.abs(model.alpha - ys / 1.08) <= 1e-8)
    # test_solver.cpp:154-167: tiny lambda nearly interpolates
    xs = np.arange(16.0)
    ys = np.sin(0.4 * xs)
    model = engine.train_krr(xs[:, None], ys, 1.0, 1e-12)
    assert np.all(np.abs(model.predict(xs[:, None]) - ys) <= 1e-4)
    assert model.residual_ratio <= 1e-8


@pytest.mark.parametrize("m,d,sigma,lam", [(100, 3, 2.0, 1e-3), (777, 90, 3.0, 1e-4), (1500, 90, 1.0, 1e-6)])
def test_train_krr_matches_oracle(engine, oracle, m, d, sigma, lam):
    X, y = mixture(m, d, 4, seed=m)
    model = engine.train_krr(X, y, sigma, lam)
    alpha, res = oracle.train_krr(X, y, sigma, lam)
    assert relnorm(model.alpha, alpha) <= REL
    assert model.residual_ratio <= 1e-8
    Q, _ = mixture(64, d, 4, seed=m + 1)
    assert relnorm(model.predict(Q), oracle.predict(X, alpha, sigma, Q)) <= REL


@pytest.mark.parametrize("m,q,d,sigma", [(1, 1, 3, 0.9), (129, 65, 7, 1.5), (20000, 1, 90, 3.0),
                                         (3000, 4100, 90, 3.0), (5000, 700, 17, 0.3)])
def test_predict_fused_matches_oracle(engine, oracle, m, q, d, sigma):
    # predict_fused.cuh: the test-by-support tile folded into the alpha contraction,
    # split over support chunks (1 .. tiles_x CTAs per query tile) and reduced in order
    rng = np.random.default_rng(m + q)
    S = rng.standard_normal((m, d))
    Q = np.vstack([S[: min(q, m) // 2], rng.standard_normal((q - min(q, m) // 2, d))])
    alpha = rng.standard_normal(m)
    got = engine.predict(S, alpha, sigma, Q)
    ref = oracle.predict(S, alpha, sigma, Q)
    # per element, relative to sum_i |K(q, i) alpha_i| <= sum |alpha| (summation-order bound)
    assert np.all(np.abs(got - ref) <= 1e-13 * np.abs(alpha).sum() + 1e-12 * np.abs(ref))
    assert np.array_equal(got, engine.predict(S, alpha, sigma, Q))  # deterministic


# ------------------------------------------------------------- clustering ----
@pytest.mark.parametrize("n,d,k,seed", [(30, 2, 1, 99), (12, 1, 12, 55), (2000, 4, 3, 17), (5000, 90, 8, 2),
                                        (9000, 90, 16, 5), (4000, 33, 40, 11), (6000, 90, 64, 13)])
def test_kmeans_bit_exact(engine, oracle, n, d, k, seed):
    X, _ = mixture(n, d, max(k, 2), seed=seed)
    g = engine.kmeans(X, k, seed)
    r = oracle.kmeans(X, k, seed)
    assert g.iterations == r["iterations"]
    assert np.array_equal(g.membership, r["membership"])
    assert np.array_equal(g.centers, r["centers"])  # order-preserving means: bitwise
    assert np.array_equal(g.sizes, r["sizes"])


def test_kmeans_forced_iterations_and_duplicates(engine, oracle):
    X, _ = mixture(3000, 90, 16, seed=4)
    g = engine.kmeans(X, 8, 7, threshold=-1.0, max_iters=20)
    r = oracle.kmeans(X, 8, 7, threshold=-1.0, max_iters=20)
    assert g.iterations == r["iterations"] == 20
    assert np.array_equal(g.membership, r["membership"]) and np.array_equal(g.centers, r["centers"])
    # duplicate points force the empty-cluster reseed path (test_clustering.cpp:100-110)
    D = np.ones((5, 2))
    g = engine.kmeans(D, 3, 8)
    r = oracle.kmeans(D, 3, 8)
    assert np.array_equal(g.membership, r["membership"]) and np.all(g.sizes >= 1)


@pytest.mark.parametrize("n,d,k,seed", [(10, 2, 3, 5), (100, 2, 2, 66), (16000, 4, 8, 2), (5003, 90, 16, 3),
                                        (777, 9, 7, 1), (3000, 90, 40, 4)])
def test_kbalance_bit_exact(engine, oracle, n, d, k, seed):
    X, _ = mixture(n, d, 4, seed=seed)
    for recompute in (True, False):
        g = engine.kbalance(X, k, seed, recompute_centers=recompute)
        r = oracle.kbalance(X, k, seed, recompute=recompute)
        assert np.array_equal(g.membership, r["membership"])
        assert np.array_equal(g.centers, r["centers"])
        assert g.sizes.max() - g.sizes.min() <= 1


def test_nearest_center_ties_and_bits(engine, oracle):
    C = np.array([[0.0], [10.0], [4.5]])
    Q = np.array([[4.5], [4.0], [5.0]])
    assert list(engine.nearest_center(C, Q)) == [2, 2, 2]
    C2 = np.array([[0.0], [10.0]])
    assert list(engine.nearest_center(C2, Q[1:])) == [0, 0]  # equidistant -> lower index
    X, _ = mixture(3000, 90, 8, seed=9)
    cen = oracle.kmeans(X, 8, 3)["centers"]
    got = engine.nearest_center(cen, X)
    want = np.array([oracle.nearest_center(cen, x) for x in X])
    assert np.array_equal(got, want)


def test_make_partition_matches_oracle(engine, oracle):
    X, _ = mixture(4000, 90, 8, seed=12)
    for kind in ("exact", "dckrr", "kkrr2", "bkrr2"):
        ps = engine.make_partition(kind, X, 4, 21)
        part, order, cen = oracle.make_partition(kind, X, 4, 21)
        got_order = np.concatenate(ps.parts)
        assert np.array_equal(got_order, order), kind
        if ps.has_centers():
            assert np.array_equal(ps.centers, cen), kind


# ------------------------------------------------------------- strategies ----
@pytest.mark.parametrize("kind", ["exact", "kkrr2", "bkrr2", "dckrr", "kkrr", "bkrr", "kkrr3", "bkrr3"])
def test_grid_search_matches_oracle(engine, oracle, kind):
    dd = datagen.make(1200, 0, 300, 12, 6, seed=3)
    lam, sig = [1e-4, 1e-2], [1.0, 3.0]
    g = engine.grid_search(kind, dd["X_train"], dd["y_train"], dd["X_test"], dd["y_test"], 4, lam, sig, 7)
    r = oracle.grid_search(kind, dd["X_train"], dd["y_train"], dd["X_test"], dd["y_test"], 4, lam, sig, 7)
    assert np.array_equal(g.failed, r["failed"])
    ok = ~r["failed"]
    assert np.all(np.abs(g.mse[ok] - r["mse"][ok]) <= REL * np.abs(r["mse"][ok]))
    assert g.best_index == r["best"]
    assert g.max_residual() <= 1e-8
    assert relnorm(g.best_pred, r["best_pred"]) <= REL


def test_train_partitions_and_predict_nearest(engine, oracle):
    dd = datagen.make(2000, 0, 200, 10, 6, seed=5)
    tp = engine.train_partitions("kkrr2", dd["X_train"], dd["y_train"], 4, 3, 2.0, 1e-4)
    part, order, cen = oracle.make_partition("kkrr2", dd["X_train"], 4, 3)
    sizes = np.bincount(part, minlength=4)
    at = 0
    for t in range(4):
        rows = order[at:at + sizes[t]]
        at += sizes[t]
        alpha, _ = oracle.train_krr(dd["X_train"][rows], dd["y_train"][rows], 2.0, 1e-4)
        assert relnorm(tp.alpha(t), alpha) <= REL
        assert tp.residual(t) <= 1e-8
    pred = tp.predict_nearest(dd["X_test"])
    from oracle import Reference
    if Reference.available():
        ref = Reference().train_predict_nearest("kkrr2", dd["X_train"], dd["y_train"], 4, 3, 2.0, 1e-4,
                                                dd["X_test"])
        assert relnorm(pred, ref) <= REL


def test_indefinite_cells_are_failed_not_fatal(engine, oracle):
    # duplicated rows make K singular; a tiny lambda then breaks the factorization
    X = np.repeat(np.linspace(0, 1, 40)[:, None], 3, axis=0)
    y = np.sin(X[:, 0])
    Q = np.linspace(0, 1, 7)[:, None]
    lam, sig = [1e-300, 1.0], [5.0]
    g = engine.grid_search("exact", X, y, Q, np.sin(Q[:, 0]), 1, lam, sig, 1)
    r = oracle.grid_search("exact", X, y, Q, np.sin(Q[:, 0]), 1, lam, sig, 1)
    assert list(g.failed) == list(r["failed"])
    assert g.best_index == r["best"]


def test_indefinite_cells_with_lookahead(engine, oracle):
    """NPD inside lookahead factorizations (parts of ~1500 rows: 12 panels > 2 groups):
    the failing slice aborts on both streams, the other cell of the part still solves,
    and the failed set / best cell equal the oracle's."""
    base = np.random.default_rng(4).uniform(-2, 2, size=(1000, 3))
    X = np.repeat(base, 3, axis=0)  # every point three times: K is singular
    y = np.sin(X[:, 0]) + X[:, 1]
    Q = np.random.default_rng(5).uniform(-2, 2, size=(64, 3))
    lam, sig = [1e-300, 1e-2], [1.5]
    g = engine.grid_search("kkrr2", X, y, Q, np.sin(Q[:, 0]) + Q[:, 1], 2, lam, sig, 3)
    r = oracle.grid_search("kkrr2", X, y, Q, np.sin(Q[:, 0]) + Q[:, 1], 2, lam, sig, 3)
    assert list(g.failed) == list(r["failed"]) == [True, False]
    assert g.best_index == r["best"] == 1
    assert abs(g.mse[1] - r["mse"][1]) <= 1e-8 * abs(r["mse"][1])
