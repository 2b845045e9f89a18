"""Regenerate tests/golden/*.npz from the REFERENCE library itself.

Runs only in the build container (needs oracle/_ref/libpkrr_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile).  The fixtures are small and committed;
tests/test_oracle.py checks the C restatement (oracle/) against them bit for bit
on any machine, so the oracle stays pinned where /root/reference is absent.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def mixture(n, d, comps, seed):
    rng = np.random.default_rng(seed)
    means = 3.0 * rng.standard_normal((comps, d))
    return means[rng.integers(0, comps, n)] + rng.standard_normal((n, d))


def main():
    r = Reference()
    g = {}
    # rng (rng.cpp)
    g["sub_seed_tags"] = np.array([r.sub_seed(s, t) for s in (0, 1, 42) for t in ("synth", "split", "partition", "sigma-grid")], np.uint64)
    g["normals_7"], g["below_7_1000"] = r.rng_stream(7, 33, 1000)
    g["perm_3_20"] = r.random_permutation(3, 20)
    # kernel (kernel.cpp)
    rng = np.random.default_rng(1)
    X = rng.standard_normal((24, 6))
    g["gram_X"] = X
    g["gram_sym_1_3"] = r.gram_sym(X, 1.3)
    Q = rng.standard_normal((5, 6))
    g["gram_Q"] = Q
    g["gram_cross_0_9"] = r.gram_cross(X, Q, 0.9)
    # solver (solver.cpp)
    G = rng.standard_normal((33, 33))
    A = G.T @ G + 16.5 * np.eye(33)
    g["spd_A"] = A
    g["chol_L"] = r.cholesky(A)
    b = rng.standard_normal(33)
    g["solve_b"] = b
    g["solve_x"] = r.solve_spd(g["chol_L"], b)
    Xk = mixture(64, 3, 3, 2)
    yk = np.sin(Xk[:, 0])
    g["krr_X"], g["krr_y"] = Xk, yk
    g["krr_alpha"], res = r.train_krr(Xk, yk, 2.0, 1e-3)
    g["krr_residual"] = np.array([res])
    Qk = mixture(9, 3, 3, 3)
    g["krr_Q"] = Qk
    g["krr_pred"] = r.train_predict(Xk, yk, 2.0, 1e-3, Qk)
    # clustering (clustering.cpp)
    Xc = mixture(400, 5, 4, 4)
    g["km_X"] = Xc
    km = r.kmeans(Xc, 4, 9)
    g["km_membership"], g["km_centers"], g["km_sizes"] = km["membership"], km["centers"], km["sizes"]
    g["km_iterations"] = np.array([km["iterations"]])
    kb = r.kbalance(Xc, 7, 9)
    g["kb_membership"], g["kb_centers"], g["kb_sizes"] = kb["membership"], kb["centers"], kb["sizes"]
    g["nearest"] = np.array([r.nearest_center(km["centers"], x) for x in Xc[:50]], np.int32)
    # strategies (strategies.cpp)
    Xt = mixture(240, 4, 5, 5)
    yt = np.cos(Xt[:, 1]) + 0.1 * Xt[:, 2]
    Xs = mixture(60, 4, 5, 6)
    ys = np.cos(Xs[:, 1]) + 0.1 * Xs[:, 2]
    g["grid_Xtr"], g["grid_ytr"], g["grid_Xte"], g["grid_yte"] = Xt, yt, Xs, ys
    g["grid_lambdas"] = np.array([1e-4, 1e-2])
    g["grid_sigmas"] = np.array([1.0, 3.0])
    for kind in ("exact", "dckrr", "kkrr", "kkrr2", "kkrr3", "bkrr", "bkrr2", "bkrr3"):
        res = r.grid_search(kind, Xt, yt, Xs, ys, 4, g["grid_lambdas"], g["grid_sigmas"], 7)
        g[f"grid_{kind}_mse"] = res["mse"]
        g[f"grid_{kind}_failed"] = res["failed"]
        g[f"grid_{kind}_residual"] = res["residual"]
        g[f"grid_{kind}_best"] = np.array([res["best"]])
        part, cen = r.make_partition(kind, Xt, 4, 7)
        g[f"part_{kind}"] = part
    # data preparation (dataset.cpp:199-232, strategies.cpp:204-234)
    rng = np.random.default_rng(8)
    Xr = 2.5 * rng.standard_normal((300, 6)) + np.arange(6)
    Xr[:, 3] = 7.0  # constant feature -> stddev 0 -> standardised to 0
    Tr = rng.standard_normal((40, 6))
    g["std_X"], g["std_T"] = Xr, Tr
    g["std_train"], g["std_test"], g["std_mean"], g["std_stddev"] = r.standardize(Xr, Tr)
    g["sigma_grid_300"] = r.auto_sigma_grid(Xr, 11)
    g["sigma_grid_700"] = r.auto_sigma_grid(mixture(700, 5, 3, 9), 11)
    g["sigma_grid_1"] = r.auto_sigma_grid(Xr[:1], 11)
    np.savez_compressed(os.path.join(OUT, "reference_vectors.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_vectors.npz"), os.path.getsize(os.path.join(OUT, "reference_vectors.npz")), "bytes")


if __name__ == "__main__":
    main()
