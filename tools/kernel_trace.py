"""Concurrent kernel timeline of one warm grid call (CUPTI activity tracing through
torch.profiler: real overlap, not the serialised ncu replay).

    python tools/kernel_trace.py [config] [--dump out.json]

Prints per-kernel totals, a 2%-bucket SM-fill estimate over the call (CTAs resident
capped at 148 per kernel, summed over overlapping kernels, capped at 1) and, for
single-part configs, the gaps on the launch stream (the panel chain)."""
import json
import os
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c1"
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
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in ev)
span = t1 - t0
print(f"{cfg}: {len(ev)} kernels, span {span / 1e3:.2f} ms")
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    nm = e["name"].split("(")[0].replace("void ", "")[:60]
    agg[nm][0] += 1
    agg[nm][1] += e["dur"]
for nm, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {d / 1e3:9.2f} ms  {n:6d}  {d / n:8.1f} us  {nm}")
nb = 50
fill = [0.0] * nb
for e in ev:
    g = e["args"].get("grid", [1, 1, 1])
    ctas = min(148, g[0] * g[1] * g[2]) / 148.0
    a, b = e["ts"] - t0, e["ts"] - t0 + e["dur"]
    for i in range(int(a * nb / span), min(nb, int(b * nb / span) + 1)):
        lo, hi = i * span / nb, (i + 1) * span / nb
        ov = max(0.0, min(b, hi) - max(a, lo))
        fill[i] += ctas * ov / (span / nb)
print("SM fill per 2% of the span:", " ".join(f"{min(1.0, f):.2f}" for f in fill))
if c["p"] == 1:
    st = defaultdict(list)
    for e in ev:
        st[e["args"].get("stream")].append(e)
    main = max(st.values(), key=len)
    gaps = [main[i + 1]["ts"] - (main[i]["ts"] + main[i]["dur"]) for i in range(len(main) - 1)]
    busy = sum(e["dur"] for e in main)
    print(f"launch stream: {len(main)} kernels, busy {busy / 1e3:.2f} ms, gaps {sum(g for g in gaps if g > 0) / 1e3:.2f} ms"
          f" (median {sorted(gaps)[len(gaps) // 2]:.1f} us)")
    for e, g in list(zip(main, gaps + [0]))[:40]:
        print(f"    {e['ts'] - t0:9.1f} +{e['dur']:7.1f} gap {g:6.1f}  {e['name'].split('(')[0][:50]}  grid {e['args'].get('grid')}")
if "--dump" in sys.argv:
    json.dump(ev, open(sys.argv[sys.argv.index("--dump") + 1], "w"))
os.unlink(path)
