import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen
eng = pk.Engine(0)
for m in [int(x) for x in sys.argv[1:]]:
    dd = datagen.make(m, 0, 0, 90, 8, seed=m)
    model = eng.train_krr(dd["X_train"], dd["y_train"], 3.0, 1e-4)
    print(m, (m + 127) // 128, "residual", model.residual_ratio, flush=True)
