"""GPU parity at BASELINE's own part sizes against the REFERENCE itself.

tests/golden/fullsize_<cfg>.npz were written by tests/golden/make_fullsize_golden.py,
which runs the unmodified reference library (oracle/_ref) at full size in the build
container (about an hour of CPU).  The inputs are regenerated here by datagen.py and
pinned by their sha256; the labels y are the fixture's own.

Covered schedules of the blocked Cholesky (csrc/kernels.cu launch_potrf): the lone
4096-row system (C0: single-panel groups, 32-row TRSM, fused forward substitution),
parts among several with G = 4 (< 8192 rows), G = 8 (8192..16383: C1's 8275 / 12298,
C2's 8192) and G = 16 (>= 16384: C1's 20544, C3's 16384), all with lookahead.

Bars (north_star): partition labels / centres bitwise; alpha, predictions and MSE
within 1e-8 relative (norm-wise for vectors).  Measured on B200: alpha within ~1e-14
of the reference on C0 / C1 / C3 and within 3.4e-12 on the worst-conditioned C2 cell
(sigma 10, lambda 1e-6).
"""
import hashlib
import os

import numpy as np
import pytest

import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    path = os.path.join(GOLD, f"fullsize_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return np.load(path)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _inputs(name, z):
    dd = datagen.config(name)
    X = dd["X_train"]
    Q = np.concatenate([dd["X_val"], dd["X_test"]]) if dd["X_val"].shape[0] else dd["X_test"]
    assert _sha(X) == str(z["x_sha"]), "datagen drift: train rows differ from the fixture's"
    assert _sha(Q) == str(z["q_sha"]), "datagen drift: query rows differ from the fixture's"
    return dd, X, Q


def test_c0_lone_system(engine):
    z = _load("c0")
    dd, X, Q = _inputs("c0", z)
    y = z["y"]
    m = engine.train_krr(X, y, 3.0, 1e-4)
    assert _rel(m.alpha, z["alpha"]) <= 1e-8, _rel(m.alpha, z["alpha"])
    assert m.residual_ratio <= 1e-8
    pred = engine.predict(X, m.alpha, 3.0, Q)
    assert _rel(pred, z["pred"]) <= 1e-8, _rel(pred, z["pred"])
    g = engine.grid_search("exact", X, y, Q, z["y_q"], 1, [1e-4], [3.0], 1)
    assert abs(g.mse[0] - float(z["mse"])) <= 1e-8 * float(z["mse"])
    assert _rel(g.best_pred, z["pred"]) <= 1e-8


def test_c1_kkrr2_every_part(engine):
    z = _load("c1")
    dd, X, Q = _inputs("c1", z)
    y = z["y"]
    km = engine.kmeans(X, 8, 1, threshold=-1.0, max_iters=20)
    assert np.array_equal(km.membership, z["membership"].astype(np.int32))
    assert km.centers.tobytes() == z["centers"].tobytes()
    assert km.iterations == int(z["iterations"]) == 20
    parts = [np.flatnonzero(km.membership == t) for t in range(8)]
    tp = engine.train_parts(X, y, parts, 3.0, 1e-4, centers=km.centers)
    at = 0
    diffs = {}
    for t in range(8):
        a = tp.alpha(t)
        ref = z["alpha"][at:at + len(a)]
        at += len(a)
        diffs[len(a)] = _rel(a, ref)
        assert _rel(a, ref) <= 1e-8, (t, len(a), _rel(a, ref))
        assert tp.residual(t) <= 1e-8
    print("C1 alpha relative difference per part size:", diffs)
    pred = tp.predict_nearest(Q)
    assert _rel(pred, z["pred"]) <= 1e-8, _rel(pred, z["pred"])
    nv = int(z["n_val"])
    # the bench's own path: one grid call, val-selected, test scored
    g = engine.grid_search("kkrr2", X, y, Q[:nv], z["y_q"][:nv], 8, [1e-4], [3.0], 1, eval_X=Q[nv:],
                           eval_y=z["y_q"][nv:], km_threshold=-1.0, km_max_iters=20)
    assert _rel(g.best_pred, z["pred"][:nv]) <= 1e-8
    assert _rel(g.best_eval_pred, z["pred"][nv:]) <= 1e-8
    assert abs(g.mse[0] - float(z["mse_val"])) <= 1e-8 * float(z["mse_val"])
    assert abs(g.eval_mse[0] - float(z["mse_test"])) <= 1e-8 * float(z["mse_test"])


def _balanced(engine, name, z, k):
    dd, X, Q = _inputs(name, z)
    kb = engine.kbalance(X, k, 1)
    assert np.array_equal(kb.membership, z["membership"].astype(np.int32))
    assert kb.centers.tobytes() == z["centers"].tobytes()
    rows = np.flatnonzero(kb.membership == 0)
    assert np.array_equal(rows, z["rows"])
    routed = np.flatnonzero(engine.nearest_center(kb.centers, Q) == 0)
    assert np.array_equal(routed, z["routed"])
    return X, Q, kb, rows, routed


def test_c3_part_16384(engine):
    """configs[3] (p = 8 step): all 8 balanced parts trained together (the bench's G = 16
    schedule among several parts); part 0 against the reference."""
    z = _load("c3")
    X, Q, kb, rows, routed = _balanced(engine, "c3", z, 8)
    y = np.zeros(X.shape[0])
    y[rows] = z["y"]
    parts = [np.flatnonzero(kb.membership == t) for t in range(8)]
    tp = engine.train_parts(X, y, parts, 3.0, 1e-5, centers=kb.centers)
    a = tp.alpha(0)
    assert len(a) == 16384
    assert _rel(a, z["alpha"][0]) <= 1e-8, _rel(a, z["alpha"][0])
    print("C3 part 0 (16384 rows) alpha relative difference:", _rel(a, z["alpha"][0]))
    pred = tp.predict(Q[routed], part=0)
    assert _rel(pred, z["pred"][0]) <= 1e-8, _rel(pred, z["pred"][0])


def test_c2_part_8192_grid(engine):
    """configs[2]: part 0 (8192 rows, the G = 8 schedule) over sigma {1,3,10} x lambda
    {1e-6,1e-4,1e-2} against the reference."""
    z = _load("c2")
    X, Q, kb, rows, routed = _balanced(engine, "c2", z, 16)
    worst = {}
    for c, (s, lam) in enumerate(z["cells"]):
        m = engine.train_krr(X[rows], z["y"], float(s), float(lam))
        pred = engine.predict(X[rows], m.alpha, float(s), Q[routed])
        worst[(s, lam)] = (_rel(m.alpha, z["alpha"][c]), _rel(pred, z["pred"][c]))
        assert m.residual_ratio <= 1e-8
        assert _rel(pred, z["pred"][c]) <= 1e-8, (s, lam, worst[(s, lam)])
        assert _rel(m.alpha, z["alpha"][c]) <= 1e-8, (s, lam, worst[(s, lam)])
    print("alpha / prediction relative differences per (sigma, lambda):", worst)
