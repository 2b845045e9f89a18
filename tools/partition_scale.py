"""k-means partition cost as the weak-scaled bench grows (n_train = 65536 N, p = 8 N,
16 N mixture components, 20 Lloyd iterations): the part every rank repeats."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402

eng = pk.Engine(0)
for N in ([int(a) for a in sys.argv[1:] if a.isdigit()] or (1, 2, 4, 8)):
    dd = datagen.make(65536 * N, 0, 0, 90, 16 * N, bumps=16, bump_sigma=3.0, clipped=False, seed=1)
    X = torch.from_numpy(dd["X_train"]).cuda()
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = eng.kmeans(X, 8 * N, 1, threshold=-1.0, max_iters=20)
        torch.cuda.synchronize()
        ms = 1e3 * (time.perf_counter() - t)
    print(f"N={N}: n={65536 * N} k={8 * N}: {ms:.1f} ms (20 iterations)", flush=True)

# the sharded partition's own compute at N = 8 (rank 0 of 8, exchange replaced by a no-op,
# so values are wrong but the per-rank kernel time is representative; add ~2 NCCL
# all-gathers + stream syncs per Lloyd iteration on a real 8-GPU node)
if "--sharded" in sys.argv:
    N = 8
    dd = datagen.make(65536 * N, 2048, 0, 90, 16 * N, bumps=16, bump_sigma=3.0, clipped=False, seed=1)
    g = {k: torch.from_numpy(v).cuda() for k, v in dd.items()}
    for label, ag in (("redundant", None), ("sharded compute, no exchange", lambda ptr, nb: None)):
        for rep in range(2):
            eng.grid_search("kkrr2", g["X_train"], g["y_train"], g["X_val"], g["y_val"], 8 * N, [1e-4], [3.0], 1,
                            km_threshold=-1.0, km_max_iters=20, rank=0, world=N, allgather=ag)
        print(f"N={N} rank 0 partition ({label}): {eng.timings()['partition']:.1f} ms", flush=True)
