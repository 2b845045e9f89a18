"""Weak-scaling bound of the bench (python tools/lpt_bound.py [c1|c3]) from its own
partitions: parts (c1: k-means, p = 8 N, 20 Lloyd iterations on n = 65536 N rows) assigned to N ranks by the engine's
LPT rule on m^3; the per-rank Cholesky load imbalance bounds the scaling efficiency
(report the attainable bound next to the measured scaling)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_1805_00569_b200 as pk  # noqa: E402
from paper_1805_00569_b200 import sharding  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
c = bench.CONFIGS[cfg]
eng = pk.Engine(0)
base = None
for N in (1, 2, 4, 8):
    dd = bench.workload(bench.CONFIGS[cfg], N)  # the bench's own weak-scaled data
    g = {k: torch.from_numpy(v).cuda() for k, v in dd.items()}
    # partition only matters here: rank 0 of N trains its parts; sizes come back for all
    thr, iters = (-1.0, c["km_iters"]) if c["km_iters"] else (0.01, 0)
    r = eng.grid_search(c["strategy"], g["X_train"], g["y_train"], g["X_val"], g["y_val"], c["p"] * N,
                        c["lambdas"], c["sigmas"], 1, km_threshold=thr, km_max_iters=iters, rank=0, world=N)
    sizes = [int(x) for x in r.parts["part_sizes"]]
    loads = [sum(float(sizes[t]) ** 3 for t in sharding.owned_parts(sizes, q, N)) for q in range(N)]
    per_rank = max(loads)
    base = base or per_rank
    print(f"N={N}: largest part {max(sizes)}, max rank load {per_rank:.3e} (mean {sum(loads) / N:.3e}): "
          f"balance {sum(loads) / N / per_rank:.3f}, weak-scaling bound vs N=1 {base / per_rank:.3f}", flush=True)
