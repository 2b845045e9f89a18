"""Lloyd k-means on the C1 training rows (65536 x 90, k = 8, exactly 20 iterations):
the assign kernel's workload, for ncu captures (e.g. -k regex:assign --launch-skip 10 -c 1)
and a CUDA-event timing of the whole k-means call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dd = datagen.config(name)
X = torch.from_numpy(dd["X_train"]).cuda()
eng = pk.Engine(0)
for _ in range(2):
    km = eng.kmeans(X, k, 1, threshold=-1.0, max_iters=20)
torch.cuda.synchronize()
s = torch.cuda.ExternalStream(eng.stream_handle)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
km = eng.kmeans(X, k, 1, threshold=-1.0, max_iters=20)
b.record(s)
b.synchronize()
print(f"kmeans {name} n={X.shape[0]} d={X.shape[1]} k={k}: {a.elapsed_time(b):.3f} ms for {km.iterations} iterations")
