"""Full-size golden fixtures from the REFERENCE library itself (BASELINE part sizes).

TEST INFRASTRUCTURE.  Runs only in the build container (needs oracle/_ref/libpkrr_ref.so,
the unmodified reference sources compiled in place by oracle/Makefile) and takes about an
hour of CPU: the reference factors a 20544-row part at ~1.5 GFLOP/s.  The GPU box cannot
run the reference at these sizes, so the -m gpu tests (tests/test_gpu_golden_fullsize.py)
compare the CUDA path with these fixtures instead.

Inputs are regenerated on any machine by datagen.py (numpy PCG64, seed 1); each fixture
stores sha256 of the train / query rows so generator drift is caught, and the labels y
themselves (so libm differences in the target's exp cannot move alpha).

Fixtures (tests/golden/fullsize_<cfg>.npz):
  c0  BASELINE configs[0]: exact KRR, one 4096-row system (the lone-system G = 1 schedule),
      sigma 3, lambda 1e-4: alpha[4096], residual, predictions of the 1024 test rows.
  c1  configs[1]: KKRR2, reference kmeans(k = 8, seed 1, threshold -1, max_iters 20) --
      exactly 20 Lloyd iterations -- membership, centres, then the reference's
      train_partitions over that partition (workers = all cores): per-part alpha (parts to
      20544 rows: G = 4/8/16 schedules), residuals, predict_nearest of val + test rows.
  c3  configs[3] (p = 8 step): kbalance(k = 8, seed 1, reference defaults) of n = 131072,
      part 0 (16384 rows) trained alone with sigma 3, lambda 1e-5; the val + test rows the
      reference routes to part 0 predicted.
  c2  configs[2]: kbalance(k = 16) of n = 131072, part 0 (8192 rows) over sigma {1,3,10} x
      lambda {1e-6,1e-4,1e-2}: alpha and routed predictions per (sigma, lambda).

    python tests/golden/make_fullsize_golden.py [c0 c1 c2 c3]
"""
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Reference  # noqa: E402
from paper_1805_00569_b200 import datagen  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CORES = os.cpu_count() or 1


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def routed(ref, centers, Q, part):
    return np.array([j for j in range(Q.shape[0]) if ref.nearest_center(centers, Q[j]) == part], np.int64)


def c0(ref):
    dd = datagen.config("c0")
    X, y, Q = dd["X_train"], dd["y_train"], dd["X_test"]
    t0 = time.perf_counter()
    alpha, res, pred, sec = ref.train_partitions_predict(X, y, np.zeros(len(X), np.int32), 1, None, 3.0, 1e-4, Q)
    wall = time.perf_counter() - t0
    np.savez_compressed(os.path.join(OUT, "fullsize_c0.npz"), x_sha=sha(X), q_sha=sha(Q), y=y, y_q=dd["y_test"],
                        sigma=3.0, lam=1e-4, alpha=alpha, residual=res, pred=pred,
                        mse=np.mean((pred - dd["y_test"]) ** 2), seconds=sec, wall=wall)
    return {"c0_wall_s": wall, "c0_part_s": sec.tolist()}


def c1(ref):
    dd = datagen.config("c1")
    X, y = dd["X_train"], dd["y_train"]
    Q = np.concatenate([dd["X_val"], dd["X_test"]])
    t0 = time.perf_counter()
    km = ref.kmeans(X, 8, 1, threshold=-1.0, max_iters=20)
    t_km = time.perf_counter() - t0
    t0 = time.perf_counter()
    alpha, res, pred, sec = ref.train_partitions_predict(X, y, km["membership"], 8, km["centers"], 3.0, 1e-4, Q,
                                                         workers=CORES)
    wall = time.perf_counter() - t0
    nv = dd["X_val"].shape[0]
    np.savez_compressed(os.path.join(OUT, "fullsize_c1.npz"), x_sha=sha(X), q_sha=sha(Q), y=y,
                        y_q=np.concatenate([dd["y_val"], dd["y_test"]]), n_val=nv, sigma=3.0, lam=1e-4,
                        membership=km["membership"].astype(np.int8), centers=km["centers"], sizes=km["sizes"],
                        iterations=km["iterations"], alpha=alpha, residual=res, pred=pred,
                        mse_val=np.mean((pred[:nv] - dd["y_val"]) ** 2),
                        mse_test=np.mean((pred[nv:] - dd["y_test"]) ** 2), seconds=sec, wall=wall)
    return {"c1_kmeans_s": t_km, "c1_train_predict_wall_s": wall, "c1_part_s": sec.tolist(),
            "c1_part_sizes": km["sizes"].tolist(), "c1_workers": CORES}


def balanced_part(ref, name, k, pool_cells):
    dd = datagen.config(name)
    X, y = dd["X_train"], dd["y_train"]
    Q = np.concatenate([dd["X_val"], dd["X_test"]])
    t0 = time.perf_counter()
    kb = ref.kbalance(X, k, 1)
    t_kb = time.perf_counter() - t0
    rows = np.flatnonzero(kb["membership"] == 0)
    tgt = routed(ref, kb["centers"], Q, 0)
    Xp, yp, Qp = X[rows], y[rows], Q[tgt]

    def cell(sl):
        s, lam = sl
        t = time.perf_counter()
        a, r, pr, _ = ref.train_partitions_predict(Xp, yp, np.zeros(len(rows), np.int32), 1, None, s, lam, Qp)
        return a, r[0], pr, time.perf_counter() - t

    with ThreadPoolExecutor(max_workers=pool_cells) as ex:
        out = list(ex.map(cell, CELLS[name]))
    return dd, X, Q, kb, rows, tgt, out, t_kb


CELLS = {"c3": [(3.0, 1e-5)], "c2": [(s, lam) for lam in (1e-6, 1e-4, 1e-2) for s in (1.0, 3.0, 10.0)]}


def cbal(ref, name, k):
    dd, X, Q, kb, rows, tgt, out, t_kb = balanced_part(ref, name, k, 9)
    yq = np.concatenate([dd["y_val"], dd["y_test"]])
    np.savez_compressed(os.path.join(OUT, f"fullsize_{name}.npz"), x_sha=sha(X), q_sha=sha(Q), k=k,
                        membership=kb["membership"].astype(np.int8), centers=kb["centers"], rows=rows.astype(np.int32),
                        y=dd["y_train"][rows], routed=tgt.astype(np.int32), y_q=yq[tgt],
                        cells=np.array(CELLS[name]), alpha=np.stack([o[0] for o in out]),
                        residual=np.array([o[1] for o in out]), pred=np.stack([o[2] for o in out]),
                        seconds=np.array([o[3] for o in out]))
    return {f"{name}_kbalance_s": t_kb, f"{name}_part_rows": int(len(rows)),
            f"{name}_cell_s": [o[3] for o in out]}


def main():
    which = sys.argv[1:] or ["c0", "c1", "c3", "c2"]
    ref = Reference()
    times = {"host_cores": CORES}
    for w in which:
        t0 = time.perf_counter()
        times.update({"c0": c0, "c1": c1}[w](ref) if w in ("c0", "c1") else cbal(ref, w, 8 if w == "c3" else 16))
        print(w, f"{time.perf_counter() - t0:.1f} s", flush=True)
    path = os.path.join(ROOT, "profiles", f"cpu_fullsize_{'_'.join(which)}_r02.json")
    with open(path, "w") as f:
        json.dump(times, f, indent=1)
    print(json.dumps(times))


if __name__ == "__main__":
    main()
