"""Host-side phase trace (PKRR_TRACE_HOST=1) of one C1 grid call with pinned HOST inputs
(the bench's e2e path) vs device-resident inputs (its `value` path)."""
import os
import sys
import time
sys.path.insert(0, ".")
os.environ["PKRR_TRACE_HOST"] = "1"
import torch  # noqa: E402
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402

dd = datagen.config("c1")
eng = pk.Engine(0)
h = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in dd.items()}
dv = {k: torch.from_numpy(v).cuda() for k, v in dd.items()}
for name, src in (("device", dv), ("host", h), ("device", dv), ("host", h)):
    t0 = time.perf_counter()
    eng.grid_search("kkrr2", src["X_train"], src["y_train"], src["X_val"], src["y_val"], 8, [1e-4], [3.0], 1,
                    eval_X=src["X_test"], eval_y=src["y_test"], km_threshold=-1.0, km_max_iters=20)
    print(f"{name}: {1e3 * (time.perf_counter() - t0):.1f} ms wall", file=sys.stderr, flush=True)
