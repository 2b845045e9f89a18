"""Seeded synthetic inputs with BASELINE.json's shapes and distributions.

The reference benchmarks on MSD / LIBSVM sets that are not available here;
BASELINE.json's configs describe synthetic stand-ins, generated here with numpy's
PCG64 (root seed recorded by the caller):
  x ~ mixture of C Gaussians (means ~ N(0, 4 I), per-cluster std 1), standardised
      with train statistics (population std);  config 4: means ~ U[0,1]^d, std 0.15,
      clipped to [0, 1], not standardised;
  y = sum_{m=1..B} a_m exp(-||x - c_m||^2 / (2 s^2)) + N(0, 0.1^2),
      a_m ~ N(0,1), c_m drawn from the train rows.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: (n_train, n_val, n_test, d, components, bumps, bump_sigma, clipped)
    "c0": (4096, 0, 1024, 90, 8, 16, 3.0, False),
    "c1": (65536, 2048, 2048, 90, 16, 16, 3.0, False),
    "c2": (131072, 2048, 2048, 90, 32, 16, 3.0, False),
    "c3": (131072, 2048, 2048, 90, 64, 16, 3.0, False),  # p=8 step of the weak-scaling sweep
    "c4": (262144, 0, 4096, 784, 10, 32, 8.0, True),
}


def make(n_train, n_val, n_test, d, comps, bumps=16, bump_sigma=3.0, clipped=False, seed=1):
    rng = np.random.default_rng(seed)
    n = n_train + n_val + n_test
    if clipped:
        means = rng.uniform(0.0, 1.0, size=(comps, d))
        comp = rng.integers(0, comps, size=n)
        X = np.clip(means[comp] + 0.15 * rng.standard_normal((n, d)), 0.0, 1.0)
    else:
        means = 2.0 * rng.standard_normal((comps, d))
        comp = rng.integers(0, comps, size=n)
        X = means[comp] + rng.standard_normal((n, d))
        mu = X[:n_train].mean(axis=0)
        sd = X[:n_train].std(axis=0)
        sd[sd == 0] = 1.0
        X = (X - mu) / sd
    centers = X[rng.integers(0, n_train, size=bumps)]
    amps = rng.standard_normal(bumps)
    d2 = (X * X).sum(1)[:, None] + (centers * centers).sum(1)[None, :] - 2.0 * X @ centers.T
    y = np.exp(-np.maximum(d2, 0.0) / (2.0 * bump_sigma ** 2)) @ amps + 0.1 * rng.standard_normal(n)
    X = np.ascontiguousarray(X)
    tr = slice(0, n_train)
    va = slice(n_train, n_train + n_val)
    te = slice(n_train + n_val, n)
    return dict(X_train=X[tr].copy(), y_train=y[tr].copy(), X_val=X[va].copy(), y_val=y[va].copy(),
                X_test=X[te].copy(), y_test=y[te].copy())


def config(name, seed=1, scale=1.0):
    n_train, n_val, n_test, d, comps, bumps, bs, clipped = CONFIGS[name]
    return make(int(n_train * scale), int(n_val * scale), int(n_test * scale), d, comps, bumps, bs, clipped, seed)
