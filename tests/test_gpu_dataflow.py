"""The dataflow Cholesky (csrc/potrf_df.cuh) that factors a system solved alone
(mp < 8192: single-part grids, pkrrgpu_cholesky / train_krr): parity with the oracle
(solver.cpp:13-72 restated), run-to-run bitwise determinism, the NPD pivot the
reference reports, and edge sizes around the 64-row tiles and 128-row padding."""
import numpy as np
import pytest

import paper_1805_00569_b200 as pk

pytestmark = pytest.mark.gpu


def gauss_spd(m, d, sigma, lam, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((m, d))
    sq = (X * X).sum(1)
    K = np.exp(-np.maximum(sq[:, None] + sq[None, :] - 2 * X @ X.T, 0) / (2 * sigma * sigma))
    return K + lam * m * np.eye(m)


@pytest.mark.parametrize("m", [1, 2, 63, 64, 65, 127, 128, 129, 700, 2049])
def test_cholesky_matches_oracle(engine, oracle, m):
    A = gauss_spd(m, 6, 1.5, 1e-3, m)
    L = engine.cholesky(A)
    R = oracle.cholesky(A)
    assert np.abs(np.triu(L, 1)).max() == 0.0
    assert np.abs(L - R).max() <= 1e-12 * np.abs(R).max()


@pytest.mark.parametrize("m", [300, 4096])
def test_factor_is_bitwise_reproducible(engine, m):
    A = gauss_spd(m, 20, 3.0, 1e-4, 7)
    L1 = engine.cholesky(A)
    L2 = engine.cholesky(A)
    assert np.array_equal(L1, L2)


# pivots at the first / last column of a 32-column panel, of a 64-column chain step,
# of a worker tile row, and deep inside the factorization
@pytest.mark.parametrize("bad", [0, 31, 32, 63, 64, 127, 700, 1499])
def test_npd_reports_the_reference_pivot(engine, oracle, bad):
    A = gauss_spd(1500, 6, 1.5, 1e-3, 3)
    A[bad, bad] = -1.0
    with pytest.raises(pk.NotPositiveDefinite) as e:
        engine.cholesky(A)
    with pytest.raises(Exception) as r:
        oracle.cholesky(A)
    assert e.value.pivot == bad == r.value.pivot
    # the engine recovers: the next call factors a good system
    L = engine.cholesky(gauss_spd(200, 6, 1.5, 1e-3, 4))
    assert np.isfinite(L).all()


@pytest.mark.parametrize("m", [129, 1000, 3000])
def test_train_krr_alpha_matches_oracle(engine, oracle, m):
    """Forward substitution inside the dataflow kernel (chain: w_k, z_k; workers: the
    L(i,k) z_k shares), backward solve over the 128-block inverses its workers form."""
    rng = np.random.default_rng(m)
    X = rng.standard_normal((m, 12))
    y = rng.standard_normal(m)
    mod = engine.train_krr(X, y, 2.0, 1e-4)
    alpha_ref, _ = oracle.train_krr(X, y, 2.0, 1e-4)
    assert np.linalg.norm(mod.alpha - alpha_ref) <= 1e-8 * np.linalg.norm(alpha_ref)
    assert mod.residual_ratio <= 1e-8


def test_fused_gram_grid_matches_separate_kernels():
    """PKRR_DF_GRAM=1 (opt-in): the dataflow kernel forms K and A = K + lambda m I tile by
    tile; the grid result must match the default path (separate gram + assemble)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, '.'); import numpy as np, paper_1805_00569_b200 as pk;"
        "from paper_1805_00569_b200 import datagen;"
        "dd = datagen.make(1500, 0, 300, 12, 4, seed=5); e = pk.Engine(0);"
        "g = e.grid_search('exact', dd['X_train'], dd['y_train'], dd['X_test'], dd['y_test'], 1,"
        " [1e-4, 1e-2], [1.5, 3.0], 1);"
        "print(repr(list(g.mse)))")
    out = {}
    for flag in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PKRR_DF_GRAM=flag),
                           capture_output=True, text=True, cwd=os.path.dirname(os.path.dirname(__file__)))
        assert r.returncode == 0, r.stderr
        out[flag] = np.array(eval(r.stdout.strip().splitlines()[-1]))
    assert np.all(np.abs(out["1"] - out["0"]) <= 1e-8 * np.abs(out["0"]))
