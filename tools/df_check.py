"""Checks / timing of the dataflow Cholesky (potrf_df.cuh) on the GPU:
factor vs numpy, determinism, NPD, train_krr vs a numpy solve, probe_potrf timing
against the stream-ordered path (PKRR_DF=0 in a subprocess).

    python tools/df_check.py [--time]
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk  # noqa: E402


def spd(m, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((m, 20))
    d2 = (X * X).sum(1)[:, None] + (X * X).sum(1)[None, :] - 2 * X @ X.T
    return np.exp(-np.maximum(d2, 0) / 18.0) + 1e-3 * m * np.eye(m)


def main():
    eng = pk.Engine(0)
    worst = 0.0
    for m in [100, 128, 200, 640, 1000, 2048, 4096, 5000, 8000]:
        A = spd(m, m)
        L = eng.cholesky(A)
        Lr = np.linalg.cholesky(A)
        err = np.abs(L - Lr).max() / np.abs(Lr).max()
        L2 = eng.cholesky(A)
        same = np.array_equal(L, L2)
        worst = max(worst, err)
        print(f"cholesky m={m}: max rel err {err:.2e}, repeat bitwise {same}", flush=True)
        assert err < 1e-12 and same, m
    # NPD
    A = spd(1000, 3)
    A[700, 700] = -1.0
    try:
        eng.cholesky(A)
        raise SystemExit("NPD not detected")
    except pk.NotPositiveDefinite as e:
        print("NPD detected, pivot", e.pivot)
    # train_krr (fused forward substitution + backward solve)
    for m in [300, 2000, 4096]:
        rng = np.random.default_rng(m)
        X = rng.standard_normal((m, 90))
        y = rng.standard_normal(m)
        mod = eng.train_krr(X, y, 3.0, 1e-4)
        K = eng.gram(X, None, 3.0)
        a = np.linalg.solve(K + 1e-4 * m * np.eye(m), y)
        err = np.linalg.norm(mod.alpha - a) / np.linalg.norm(a)
        print(f"train_krr m={m}: alpha rel err {err:.2e}, residual {mod.residual_ratio:.2e}", flush=True)
        assert err < 1e-10
    if "--time" in sys.argv:
        for m in [2048, 4096, 8000]:
            for _ in range(2):
                eng.probe_potrf(m, alone=True)
            r = min((eng.probe_potrf(m, alone=True) for _ in range(5)), key=lambda r: r["total_ms"])
            out = subprocess.run([sys.executable, "-c",
                                  "import sys; sys.path.insert(0,'.'); import paper_1805_00569_b200 as pk; e=pk.Engine(0);"
                                  f"[e.probe_potrf({m}, True) for _ in range(2)];"
                                  f"print(min(e.probe_potrf({m}, True)['total_ms'] for _ in range(5)))"],
                                 env=dict(os.environ, PKRR_DF="0"), capture_output=True, text=True)
            print(f"potrf m={m} alone: dataflow {r['total_ms']:.3f} ms "
                  f"({r['chol_flops'] / r['total_ms'] / 1e9:.1f} TFLOP/s), stream-ordered {out.stdout.strip()} ms",
                  flush=True)


if __name__ == "__main__":
    main()
