"""C1 grid once: per-part system residuals and the selection MSE (any PKRR_* mode,
e.g. PKRR_SYRK=ozaki or PKRR_SHADOW=1)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen
dd = datagen.config("c1")
eng = pk.Engine(0)
res = eng.grid_search("kkrr2", dd["X_train"], dd["y_train"], dd["X_val"], dd["y_val"], 8, [1e-4], [3.0], 1,
                      km_threshold=-1.0, km_max_iters=20)
print("part residuals", ["%.1e" % x for x in res.parts["part_residual"][0]], "mse", res.mse[0])
