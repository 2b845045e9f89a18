"""Kernel timeline of the END of one warm grid call (CUPTI through torch.profiler): every
kernel that starts after the last Cholesky kernel of the call ends, per stream -- what runs
between the end of the factorizations and the end of the step.

    python tools/tail_trace.py [config]
"""
import json
import os
import sys
import tempfile

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
c = bench.CONFIGS[cfg]
dd = datagen.config(cfg)
eng = pk.Engine(0)
dv = {k: torch.from_numpy(v).cuda() for k, v in dd.items()}
if c["val"]:
    sX, sy, kw = dv["X_val"], dv["y_val"], dict(eval_X=dv["X_test"], eval_y=dv["y_test"])
else:
    sX, sy, kw = dv["X_test"], dv["y_test"], {}
if c.get("km_iters"):
    kw.update(km_threshold=-1.0, km_max_iters=c["km_iters"])


def call():
    return eng.grid_search(c["strategy"], dv["X_train"], dv["y_train"], sX, sy, c["p"], c["lambdas"], c["sigmas"],
                           1, **kw)


for _ in range(3):
    call()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    call()
    torch.cuda.synchronize()
path = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
os.unlink(path)
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in ev)
chol = ("dsyrk", "potrf", "dgemm_tn", "trsm")
last_chol = max(e["ts"] + e["dur"] for e in ev if any(k in e["name"] for k in chol))
print(f"{cfg}: span {(t1 - t0) / 1e3:.2f} ms, last Cholesky kernel ends at {(last_chol - t0) / 1e3:.2f} ms")
first = [e for e in ev if e["ts"] - t0 < 7000]
print("first 7 ms: per kernel totals")
agg = {}
for e in first:
    nm = e["name"].split("(")[0].replace("void ", "")[:50]
    a = agg.setdefault(nm, [0, 0.0])
    a[0] += 1
    a[1] += e["dur"]
for nm, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {d / 1e3:8.3f} ms {n:5d}  {nm}")
busy = 0.0
cur = None
for e in first:
    a, b = e["ts"], e["ts"] + e["dur"]
    if cur is None or a > cur:
        busy += b - a
        cur = b
    elif b > cur:
        busy += b - cur
        cur = b
print(f"  union of kernel intervals in the first 7 ms: {busy / 1e3:.2f} ms")
print("tail (kernels ending within 9 ms of the end):")
for e in ev:
    if e["ts"] + e["dur"] > t1 - 9000 and e["dur"] > 30:
        print(f"  {(e['ts'] - t0) / 1e3:9.3f} +{e['dur'] / 1e3:7.3f} ms  stream {e['args'].get('stream')}  "
              f"{e['name'].split('(')[0].replace('void ', '')[:44]}  grid {e['args'].get('grid')}")
