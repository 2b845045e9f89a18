"""Repeated C1 grid calls (all the concurrency: part streams, lookahead companions,
programmatic dependent launch, the residual on a side stream): predictions, MSE and
residuals must be bitwise identical every time."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dd = datagen.config("c1")
g = {k: torch.from_numpy(v).cuda() for k, v in dd.items()}
eng = pk.Engine(0)
ref = None
bad = 0
for i in range(reps):
    r = eng.grid_search("kkrr2", g["X_train"], g["y_train"], g["X_val"], g["y_val"], 8, [1e-4], [3.0], 1,
                        eval_X=g["X_test"], eval_y=g["y_test"], km_threshold=-1.0, km_max_iters=20)
    sig = (r.best_pred.tobytes(), r.mse.tobytes(), r.parts["part_residual"].tobytes())
    if ref is None:
        ref = sig
    elif sig != ref:
        bad += 1
print(f"{reps} C1 grid calls: {bad} differ from the first (max residual {r.parts['part_residual'].max():.2e})")
sys.exit(1 if bad else 0)
