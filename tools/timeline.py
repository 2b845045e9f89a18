"""Per-part timeline of one grid call (first cell): gram, Cholesky, solve/predict.

    python tools/timeline.py [config]      (PKRR_* env knobs apply)
"""
import sys

sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
c = bench.CONFIGS[cfg]
dd = datagen.config(cfg)
eng = pk.Engine(0)
if c["val"]:
    sX, sy, kw = dd["X_val"], dd["y_val"], dict(eval_X=dd["X_test"], eval_y=dd["y_test"])
else:
    sX, sy, kw = dd["X_test"], dd["y_test"], {}
if c.get("km_iters"):
    kw.update(km_threshold=-1.0, km_max_iters=c["km_iters"])
for _ in range(3):
    r = eng.grid_search(c["strategy"], dd["X_train"], dd["y_train"], sX, sy, c["p"], c["lambdas"], c["sigmas"], 1,
                        want_partition=True, **kw)
t = eng.timings(c["p"])
print(f"{cfg}: total {t['total']:.1f} ms, partition {t['partition']:.1f}, chol(union) {t['cholesky']:.1f}, "
      f"gram(union) {t['gram']:.1f}, predict(union) {t['predict']:.1f}")
sizes = r.parts["part_sizes"]
for q, tl in enumerate(t["part_timeline_ms"]):
    g0, g1, c0, c1, p1 = tl
    m = int(sizes[q])
    print(f"  part {q:2d} m={m:6d}: gram {g0:7.1f}-{g1:7.1f}  chol {c0:7.1f}-{c1:7.1f} ({c1 - c0:6.1f})  "
          f"solve+pred -> {p1:7.1f} ({p1 - c1:5.1f})")
