"""Small end-to-end exercise of every kernel for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen

eng = pk.Engine(0)
dd = datagen.make(700, 40, 40, 12, 4, seed=2)
for kind in ("exact", "kkrr2", "bkrr2", "dckrr", "kkrr3"):
    eng.grid_search(kind, dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"], 3, [1e-4, 1e-2], [1.0, 3.0], 1,
                    eval_X=dd["X_test"], eval_y=dd["y_test"])
X = dd["X_train"][:300]
L = eng.cholesky(eng.gram(X, X, 2.0) + 0.1 * np.eye(300))
eng.solve_spd(L, np.ones(300))
eng.kbalance(dd["X_train"], 5, 3)
tp = eng.train_partitions("kkrr2", dd["X_train"], dd["y_train"], 3, 1, 2.0, 1e-3)
tp.predict_nearest(dd["X_test"])
print("sanitize probe ok")
