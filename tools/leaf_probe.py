"""Small driver for profiling the Cholesky leaf / SYRK kernels in isolation."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
rng = np.random.default_rng(0)
X = rng.standard_normal((m, 90))
y = rng.standard_normal(m)
eng = pk.Engine(0)
for _ in range(2):
    eng.train_krr(X, y, 3.0, 1e-4)
print("ok", m)
