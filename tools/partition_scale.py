"""k-means partition cost as the weak-scaled bench grows (n_train = 65536 N, p = 8 N,
16 N mixture components, 20 Lloyd iterations): the part every rank repeats."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402

eng = pk.Engine(0)
for N in ([int(a) for a in sys.argv[1:]] or (1, 2, 4, 8)):
    dd = datagen.make(65536 * N, 0, 0, 90, 16 * N, bumps=16, bump_sigma=3.0, clipped=False, seed=1)
    X = torch.from_numpy(dd["X_train"]).cuda()
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = eng.kmeans(X, 8 * N, 1, threshold=-1.0, max_iters=20)
        torch.cuda.synchronize()
        ms = 1e3 * (time.perf_counter() - t)
    print(f"N={N}: n={65536 * N} k={8 * N}: {ms:.1f} ms (20 iterations)", flush=True)
