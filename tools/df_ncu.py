"""One m x m lone factorization through the library (the dataflow kernel), for ncu."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(0)
X = rng.standard_normal((m, 20))
sq = (X * X).sum(1)
A = np.exp(-np.maximum(sq[:, None] + sq[None, :] - 2 * X @ X.T, 0) / 18.0) + 1e-3 * m * np.eye(m)
eng = pk.Engine(0)
for _ in range(2):
    L = eng.cholesky(A)
print("ok", m, float(np.abs(L).max()))
