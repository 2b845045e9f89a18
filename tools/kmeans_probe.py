"""Driver for profiling the partition (k-means, 20 forced Lloyd iterations) on the C1 shape."""
import sys
import time
sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import datagen

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dd = datagen.make(65536, 0, 0, 90, 16, seed=1)
eng = pk.Engine(0)
import torch
X = torch.from_numpy(dd["X_train"]).cuda()
for _ in range(3):
    t0 = time.perf_counter()
    c = eng.kmeans(X, k, 1, threshold=-1.0, max_iters=20)
    print("kmeans wall ms", 1e3 * (time.perf_counter() - t0), c.iterations, c.sizes)
