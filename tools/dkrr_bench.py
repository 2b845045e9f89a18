"""DKRR (one exact system factorised across a GPU group, csrc/dist.cu) against the
one-GPU exact path, on one B200: wall time of train_krr (gram + Cholesky + solves +
residual) and the Cholesky count m(m+1)(2m+1)/6 per second.

  python tools/dkrr_bench.py [m ...]      (default 16384 32768)
Groups: [0] (the distributed code with one GPU: its per-GPU efficiency) and [0, 0]
(two contexts sharing the GPU: the exchange / chain overhead; no speed-up possible)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402


def timed(fn, reps=2):
    fn()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        best = min(best, time.perf_counter() - t0)
    return best, out


sizes = [int(a) for a in sys.argv[1:]] or [16384, 32768]
eng = pk.Engine(0)
g1, g2 = pk.Group([0]), pk.Group([0, 0])
rows = []
for m in sizes:
    dd = datagen.make(m, 0, 8, 90, 16, seed=7)
    X, y = dd["X_train"], dd["y_train"]
    flops = m * (m + 1) * (2 * m + 1) / 6
    t_one, mod = timed(lambda: eng.train_krr(X, y, 3.0, 1e-4))
    t_d1, (a1, r1) = timed(lambda: g1.train_krr(X, y, 3.0, 1e-4))
    t_d2, (a2, r2) = timed(lambda: g2.train_krr(X, y, 3.0, 1e-4))
    rel = lambda a: float(np.linalg.norm(a - mod.alpha) / np.linalg.norm(mod.alpha))  # noqa: E731
    row = dict(m=m, one_gpu_s=t_one, dkrr_w1_s=t_d1, dkrr_w2_same_gpu_s=t_d2,
               one_gpu_tflops=flops / t_one / 1e12, dkrr_w1_tflops=flops / t_d1 / 1e12,
               dkrr_w2_tflops=flops / t_d2 / 1e12, alpha_rel_w1=rel(a1), alpha_rel_w2=rel(a2),
               residual_w1=r1, residual_w2=r2)
    rows.append(row)
    print(json.dumps(row), flush=True)
