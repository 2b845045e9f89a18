#!/usr/bin/env python
"""Benchmark of the partitioned Gaussian KRR hot path (BASELINE.json configs[1]).

Default workload ("step"):
  N = 1: BASELINE configs[1] (--config c1) -- KKRR2, synthetic (datagen.py, seed 1):
      n_train = 65536, n_val = 2048, n_test = 2048, d = 90, 16-component mixture; Lloyd
      k-means into p = 8 parts (exactly 20 iterations), one Gaussian KRR model per part
      (sigma 3, lambda 1e-4: gram + lambda*m_t*I + Cholesky + solves + residual), val and
      test rows routed to the nearest centroid's model, MSE, best cell selected on
      validation MSE.
  N > 1: BASELINE configs[3] (--config c3), the reference's weak-scaling config -- BKRR2
      with 16384 rows per part and p = 8 N parts (n_train = 131072 N), sigma 3,
      lambda 1e-5; parts sharded by LPT on m^3 with no data-path collective, the ranks'
      per-cell predictions summed (disjoint) and combined once.
--config c0|c1|c2|c3|c4 picks a config explicitly (CONFIGS): c1 / c3 scale n and p
with N (weak), c2 keeps its 16 parts of 8192 rows over N GPUs (strong), c0 / c4 are
single-GPU configs.  `--gpus N` without torchrun re-launches this script under
torch.distributed.run with N ranks (and fails if fewer than N GPUs are visible).

Metric: train+predict samples/s = (n_train + n_val + n_test) * cells / step time.
`value` times the engine with inputs resident in HBM (CUDA events on the engine's
launch stream, L2 flushed between steps); `e2e` times the public API with pinned
HOST buffers (H2D of inputs and D2H of results inside the timed region).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context (see pkrrgpu_create)

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train+predict samples/sec (FP64)"
# DRAM bytes (read, write) and 128x128 tiles of one trailing-SYRK launch per K, from the
# committed ncu --set full captures of the m = 20544 factorization probe:
# K=2048 profiles/ncu_syrk_k2048_r02.txt (banded tile order, round 2; K=1024 / K=512 from the
# metrics-only pass noted there);
# K=128 (a lone 4096-row system, C0): ncu_syrk_k128_r01.txt (tools/syrk_probe_alone.py).
# DRAM bytes (read, write) of the dataflow Cholesky's ncu capture (m = 4096 lone system,
# profiles/ncu_df_c0_r02b.txt)
DF_NCU_BYTES = {4096: (73.19e6, 56.23e6)}


def DF_ROOFLINE(m, tflops, peak, probe):
    """Roofline object for a lone system factorised by the dataflow kernel: the whole
    factorization is one launch; achieved = the reference's Cholesky flop count
    m(m+1)(2m+1)/6 (solver.cpp:39-42) / that launch's duration (probe_potrf, CUDA events)."""
    nb = DF_NCU_BYTES.get(m)
    return {"bound": "tensor",
            "kernel": "potrf_df_kernel (the whole Cholesky of the lone system: chain CTA + 147 DMMA worker CTAs)",
            "achieved": tflops, "peak": peak, "unit": "TFLOP/s", "frac": tflops / peak if peak else None,
            "traffic": (nb[0] + nb[1]) if nb else None,
            "traffic_note": ("DRAM read+write bytes of the captured launch (ncu --set full, profiles/ncu_df_c0_r02b.txt) "
                             "vs 4 m^2 = 67 MB of lower-triangle operands: the matrix stays L2-resident (hit 91.8 %)"
                             if nb else "no ncu capture for this m"),
            "peak_source": "measured live after the warm-up, best of 3: FP64 DMMA (mma.sync m8n8k4) probe over "
                           "148 SMs; MEASURED_PEAKS.json has no FP64 entry",
            "algorithmic": f"m(m+1)(2m+1)/6 for m={m} / the launch's event-timed duration "
                           f"({probe['total_ms']:.3f} ms, standalone factorization)"}


SYRK_NCU_LAUNCH = {128: (351, 49.44e6, 1.77e6), 512: (11781, 2.26e9, 1.51e9), 1024: (11781, 3.18e9, 1.53e9),
                   2048: (10585, 6.10e9, 1.38e9)}
UNIT = "samples/s"


def syrk_traffic_note(k):
    """DRAM bytes of the captured trailing-SYRK launch against (a) its compulsory bytes --
    every lower C tile read and written once, the panel read once -- and (b) the no-reuse
    figure where every tile fetches its own operands from HBM."""
    if k not in SYRK_NCU_LAUNCH:
        return "no ncu capture for this K"
    tiles, rd, wr = SYRK_NCU_LAUNCH[k]
    rows = 128 * ((-1 + (1 + 8 * tiles) ** 0.5) / 2)  # tiles = T (T + 1) / 2 lower tiles
    compulsory = tiles * 2 * 128 * 128 * 8 + rows * k * 8
    no_reuse = tiles * (2 * 128 * k * 8 + 2 * 128 * 128 * 8)
    return (f"DRAM read+write bytes of the captured K={k} launch ({tiles} tiles of 128x128, ncu --set full, "
            f"profiles/): {(rd + wr) / compulsory:.1f}x its compulsory {compulsory:.3e} B (each lower C tile read and "
            f"written once, the panel once) and {(rd + wr) / no_reuse:.2f}x the no-reuse {no_reuse:.3e} B (tiles run in "
            "bands of 8 tile rows and blocks of 8 tile columns, so the panel rows in flight stay in L2; row-major order took 5.7x the compulsory "
            "bytes at K=2048); the launch is DMMA-bound (tensor pipe 88-94 % in the captures), not HBM-bound")

# BASELINE.json configs (per GPU for the weak-scaled ones).  km_iters 20 = exactly
# 20 Lloyd iterations (threshold -1); 0 = the reference defaults (0.01 / 100).
CONFIGS = {
    "c0": dict(name="configs[0]: exact KRR, one part", strategy="exact", n=4096, val=0, test=1024, d=90, comps=8,
               p=1, sigmas=[3.0], lambdas=[1e-4], bump=3.0, clipped=False, km_iters=0, scale_n=False),
    "c1": dict(name="configs[1]: KKRR2, k-means(20 it) p=8, val-selected", strategy="kkrr2", n=65536, val=2048,
               test=2048, d=90, comps=16, p=8, sigmas=[3.0], lambdas=[1e-4], bump=3.0, clipped=False, km_iters=20,
               scale_n=True),
    "c2": dict(name="configs[2]: BKRR2, k-balance p=16, 3 sigma x 3 lambda", strategy="bkrr2", n=131072, val=2048,
               test=2048, d=90, comps=32, p=16, sigmas=[1.0, 3.0, 10.0], lambdas=[1e-6, 1e-4, 1e-2], bump=3.0,
               clipped=False, km_iters=0, scale_n=False),
    "c3": dict(name="configs[3]: weak-scaling BKRR2, 16384 rows/part, p=8 per GPU", strategy="bkrr2", n=131072,
               val=2048, test=2048, d=90, comps=64, p=8, sigmas=[3.0], lambdas=[1e-5], bump=3.0, clipped=False,
               km_iters=0, scale_n=True, scale_comps=False),
    "c4": dict(name="configs[4]: wide-feature KKRR2, d=784, p=8", strategy="kkrr2", n=262144, val=0, test=4096,
               d=784, comps=10, p=8, sigmas=[8.0], lambdas=[1e-4], bump=8.0, clipped=True, km_iters=0,
               scale_n=False),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sample-n", type=int, default=0, help="reference sample train rows (0 = auto)")
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c1 at N = 1, c3 (the weak-scaling config) at N > 1")
    ap.add_argument("--update", default="fp64", choices=["fp64", "int8"],
                    help="trailing Cholesky update: FP64 tensor cores (DMMA, default) or the opt-in "
                         "FP64-accurate int8 Ozaki emulation (tcgen05 kind::i8)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload(cfg, world):
    from paper_1805_00569_b200 import datagen
    mult = world if cfg["scale_n"] else 1
    comps = cfg["comps"] * (mult if cfg.get("scale_comps", True) else 1)
    return datagen.make(cfg["n"] * mult, cfg["val"], cfg["test"], cfg["d"], comps,
                        bumps=32 if cfg["clipped"] else 16, bump_sigma=cfg["bump"], clipped=cfg["clipped"], seed=1)


def selection(dd):
    """(selection X, y, eval X, y): val selects and test is scored when there is a
    validation split; otherwise test selects (the reference's grid_search semantics)."""
    if dd["X_val"].shape[0]:
        return dd["X_val"], dd["y_val"], dd["X_test"], dd["y_test"]
    return dd["X_test"], dd["y_test"], None, None


# ---------------------------------------------------------------- clocks ----
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.gpu = gpu

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ reference ----
def reference_sample(cfg, dd, n_s, workers):
    """Time the UNMODIFIED reference (oracle/_ref, compiled from /root/reference
    sources) through its own grid_search on a bounded sample of the workload: the
    first n_s train rows (same generator), the config's strategy, p and grid, all
    val+test rows as its (selection) test set."""
    from oracle import Reference
    ref = Reference()
    Xs, ys = dd["X_train"][:n_s], dd["y_train"][:n_s]
    Xq = np.concatenate([dd["X_val"], dd["X_test"]])
    yq = np.concatenate([dd["y_val"], dd["y_test"]])
    t0 = time.perf_counter()
    r = ref.grid_search(cfg["strategy"], Xs, ys, Xq, yq, cfg["p"], cfg["lambdas"], cfg["sigmas"], 1,
                        workers=workers)
    dt = time.perf_counter() - t0
    return r, dt, (Xs, ys, Xq, yq)


def _lpt_makespan(costs, workers):
    """run_partitions (runtime.hpp:70-112) hands parts to `workers` threads in index
    order as they free up; the makespan of that list schedule."""
    import heapq
    free = [0.0] * max(1, min(workers, len(costs)))
    for c in costs:
        t = heapq.heappop(free)
        heapq.heappush(free, t + c)
    return max(free)


# Reference CPU cost of one part's train + predict vs its size: T ~ m^3.31, fitted to the
# reference's own full-size runs (tests/golden/make_fullsize_golden.py, profiles/
# cpu_fullsize_*_r02.json: m = 4096 in 8.3 s, m = 20544 in 1740 s on one core each).  The
# exponent is above 3 because the reference's unblocked Cholesky falls out of cache as m
# grows (1.75 GFLOP/s at m = 4096 down to 1.66 at 20544 per core).
CPU_COST_EXP = 3.31


def cpu_extrapolation(cfg, dd, n_s, workers):
    """Full-size / sample CPU-time ratio of the reference grid: each part costs
    cells * m^CPU_COST_EXP, the parts are scheduled over `workers` threads like
    run_partitions (runtime.hpp:70-112, index order), and the parts come from the
    reference's own make_partition of the sample and of the full training set.
    Checked against the measured full-size C1 run (profiles/cpu_fullsize_c1_r02.json)."""
    from oracle import Reference
    ref = Reference()
    ncell = len(cfg["sigmas"]) * len(cfg["lambdas"])

    def makespan(X):
        part, _ = ref.make_partition(cfg["strategy"], X, cfg["p"], 1)
        sizes = np.bincount(part).astype(float)
        return _lpt_makespan([ncell * m ** CPU_COST_EXP for m in sizes], workers), sizes

    full, fs = makespan(dd["X_train"])
    samp, ss = makespan(dd["X_train"][:n_s])
    return full / samp, [int(x) for x in fs], [int(x) for x in ss]


def sample_rows(cfg, steps, warmup, override):
    """Bounded CPU sample: parts of ~2048 rows (1024 for multi-cell grids), so one
    reference step is a few seconds on the host's cores."""
    if override:
        return override
    per_part = 2048 if len(cfg["sigmas"]) * len(cfg["lambdas"]) == 1 else 1024
    if steps + warmup > 30 or cfg["d"] > 200:
        per_part //= 2
    return min(cfg["n"], per_part * cfg["p"])


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    dd = workload(cfg, 1)
    cores = os.cpu_count() or 1
    n_s = sample_rows(cfg, args.steps, args.warmup, args.sample_n)
    for _ in range(args.warmup):
        reference_sample(cfg, dd, n_s, cores)
    times = []
    for _ in range(args.steps):
        _, dt, _ = reference_sample(cfg, dd, n_s, cores)
        times.append(dt)
    ms = 1e3 * statistics.mean(times)
    ncell = len(cfg["sigmas"]) * len(cfg["lambdas"])
    samples = (n_s + cfg["val"] + cfg["test"]) * ncell
    value = samples / (ms / 1e3)
    sample = (f"first {n_s} of {cfg['n']} train rows, {cfg['strategy']} p={cfg['p']} (parts ~{n_s // cfg['p']} rows "
              f"vs ~{cfg['n'] // cfg['p']} at full size), {ncell} cell(s), {cfg['val'] + cfg['test']} val+test "
              f"rows; reference grid_search with GridOptions.workers={cores}")
    ratio, full_sizes, sample_sizes = cpu_extrapolation(cfg, dd, n_s, cores)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if cfg["scale_n"] else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"BASELINE {cfg['name']} (bounded CPU sample)", "n_train_sample": n_s,
                       "n_train": cfg["n"], "n_val": cfg["val"], "n_test": cfg["test"], "d": cfg["d"],
                       "p": cfg["p"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample,
                             "extrapolated_full_value": value * (cfg["n"] + cfg["val"] + cfg["test"])
                             / (n_s + cfg["val"] + cfg["test"]) / ratio,
                             "extrapolation": "sample time x (full / sample) makespan of per-part reference "
                                              "costs m^3.31 over the cores (bench.cpu_extrapolation); measured "
                                              "full-size C1 reference: 1749 s on 8 cores "
                                              "(profiles/cpu_fullsize_c1_r02.json)",
                             "full_part_sizes": full_sizes, "sample_part_sizes": sample_sizes},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def full_size_parity(name, eng, dd):
    """alpha / prediction / MSE agreement with the REFERENCE at the workload's full size:
    the reference's own outputs (tests/golden/fullsize_<cfg>.npz, written by
    tests/golden/make_fullsize_golden.py from oracle/_ref; the box cannot run it at this
    size in minutes) against this engine on the same regenerated inputs."""
    import hashlib
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz")
    if name not in ("c0", "c1") or not os.path.exists(path):
        return {"unavailable": f"no full-size fixture for {name}"}
    z = np.load(path)
    X = dd["X_train"]
    Q = np.concatenate([dd["X_val"], dd["X_test"]])
    if hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest() != str(z["x_sha"]):
        return {"unavailable": "datagen drift"}
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    if name == "c0":
        m = eng.train_krr(X, z["y"], 3.0, 1e-4)
        pred = eng.predict(X, m.alpha, 3.0, Q)
        mse = float(np.mean((pred - z["y_q"]) ** 2))
        return {"reference": f"oracle/_ref at full size (tests/golden/fullsize_c0.npz, {float(z['wall']):.1f} s)",
                "alpha_max_rel_diff": rel(m.alpha, z["alpha"]), "pred_rel_diff": rel(pred, z["pred"]),
                "mse_rel_diff": abs(mse - float(z["mse"])) / float(z["mse"])}
    km = eng.kmeans(X, 8, 1, threshold=-1.0, max_iters=20)
    parts = [np.flatnonzero(km.membership == t) for t in range(8)]
    tp = eng.train_parts(X, z["y"], parts, 3.0, 1e-4, centers=km.centers)
    at, worst = 0, 0.0
    for t in range(8):
        a = tp.alpha(t)
        worst = max(worst, rel(a, z["alpha"][at:at + len(a)]))
        at += len(a)
    pred = tp.predict_nearest(Q)
    nv = int(z["n_val"])
    mse_v = float(np.mean((pred[:nv] - z["y_q"][:nv]) ** 2))
    return {"reference": "oracle/_ref at full size (tests/golden/fullsize_c1.npz, 1749 s on 8 cores)",
            "labels_bitwise": bool(np.array_equal(km.membership, z["membership"].astype(np.int32))),
            "alpha_max_rel_diff": worst, "pred_rel_diff": rel(pred, z["pred"]),
            "mse_val_rel_diff": abs(mse_v - float(z["mse_val"])) / float(z["mse_val"])}


# -------------------------------------------------------------------- ours ----
def run_ours(args):
    import torch
    import paper_1805_00569_b200 as pk

    cfg = CONFIGS[args.config]
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    dd = workload(cfg, world)
    mult = world if cfg["scale_n"] else 1
    n_train = cfg["n"] * mult
    p = cfg["p"] * mult if cfg["p"] > 1 else 1
    ncell = len(cfg["sigmas"]) * len(cfg["lambdas"])
    eng = pk.Engine(local)
    stream = torch.cuda.ExternalStream(eng.stream_handle, device=dev)

    g = {k: torch.from_numpy(v).to(dev) for k, v in dd.items()}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    thr, iters = (-1.0, cfg["km_iters"]) if cfg["km_iters"] else (0.01, 0)
    # the partition (every rank needs it) is sharded over the ranks from N = 4 on: rows'
    # assignments and whole clusters' centroid chains split, NCCL all-gathers per Lloyd
    # iteration, bitwise the single-process partition (sharding.torch_allgather); below
    # that the redundant partition is as fast (tools/partition_scale.py)
    shard_env = os.environ.get("PKRR_SHARD_PARTITION")
    shard = world > 1 and (world >= 4 if shard_env is None else shard_env == "1")
    allgather = None
    if shard:
        from paper_1805_00569_b200 import sharding
        allgather = sharding.torch_allgather(dist, rank, world, dev)

    def step(src):
        sX, sy, eX, ey = selection(src)
        return eng.grid_search(cfg["strategy"], src["X_train"], src["y_train"], sX, sy, p, cfg["lambdas"],
                               cfg["sigmas"], 1, eval_X=eX, eval_y=ey, km_threshold=thr, km_max_iters=iters,
                               rank=rank, world=world, allgather=allgather)

    for _ in range(args.warmup):
        step(g)
    torch.cuda.synchronize(dev)
    # FP64 DMMA peak of this GPU, measured warm (after the warm-up steps), best of 3: a
    # stable (upper) roofline denominator
    peak = max(eng.fp64_peak() for _ in range(3))
    if world > 1:
        dist.barrier()
    clk = Clocks(local)
    clk.start()
    t_wall0 = time.perf_counter()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = eng.launches
    phase = {"chol": 0.0, "gram": 0.0, "partition": 0.0, "total": 0.0}
    flops = {"chol": 0.0, "gram": 0.0, "other": 0.0}
    res = None
    t = {}
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            res = step(g)
            ev[i][1].record(stream)
            t = eng.timings(parts=res.p)
            phase["chol"] += t["cholesky"]
            phase["gram"] += t["gram"]
            phase["partition"] += t["partition"]
            phase["total"] += t["total"]
            for k in flops:
                flops[k] += res.flops[k]
    torch.cuda.synchronize(dev)
    launches = eng.launches - l0
    # a timed region shorter than nvidia-smi's sampling period (C0: 5 steps of 2 ms) would
    # leave no clock sample: keep the same step running, untimed, until ~1 s has passed
    extended = 0
    t_clk = time.perf_counter()
    # (one rank only: with several ranks a time-based loop would run different numbers of
    # steps -- and of their collectives -- on different ranks; those runs are longer than 1 s)
    while world == 1 and time.perf_counter() - t_wall0 < 1.0 and time.perf_counter() - t_clk < 1.5:
        with torch.cuda.stream(stream):
            step(g)
        torch.cuda.synchronize(dev)
        extended += 1
    clocks = clk.stop()
    if extended:
        clocks["note"] = f"timed region < 1 s: sampling continued over {extended} more untimed steps of the same workload"
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.mean(step_ms)
    n_sel = cfg["val"] if cfg["val"] else cfg["test"]
    n_eval = cfg["test"] if cfg["val"] else 0
    # --- multi-rank: max time over ranks, part-order combine of per-part SSE ---
    if world > 1:
        from paper_1805_00569_b200 import sharding
        tms = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        ms = float(tms.item())
        parts = res.parts
        sX, sy, eX, ey = selection(dd)
        pred, fcell = sharding.allreduce_predictions(parts["cell_pred"], parts["part_failed"], dist, device=dev)
        sel_mse, best, _ = sharding.combine(eng, cfg["strategy"], p, pred, fcell, sy)
        if n_eval:
            epred, _ = sharding.allreduce_predictions(parts["cell_eval_pred"], parts["part_failed"], dist, device=dev)
            eval_mse, _, _ = sharding.combine(eng, cfg["strategy"], p, epred, fcell, ey)
        else:
            eval_mse = sel_mse
    else:
        sel_mse, best = res.mse, res.best_index
        eval_mse = res.eval_mse if n_eval else res.mse
    samples = (n_train + cfg["val"] + cfg["test"]) * ncell
    value = samples / (ms / 1e3)
    chol_tflops = flops["chol"] / (phase["chol"] / 1e3) / 1e12 if phase["chol"] > 0 else 0.0
    step_tflops = (flops["chol"] + flops["gram"] + flops["other"]) / (sum(step_ms) / 1e3) / 1e12

    # --- dominant kernel, live: the largest part's factorization alone on one stream,
    # CUDA events around every trailing-SYRK launch (algorithmic flops / launch time)
    big = int(max(res.parts["part_sizes"]))
    nb_big = (big + 127) // 128  # the library's automatic panel group (kernels.cu launch_potrf)
    alone = len(res.parts["part_sizes"]) == 1  # a lone small system: single-panel groups
    ozaki = os.environ.get("PKRR_SYRK") == "ozaki"
    syrk_k = (128 if alone and not ozaki else 512) if (nb_big < 64 or ozaki) else (1024 if nb_big < 128 else 2048)
    # best of 3 (the first call builds the dataflow task list / workspace)
    probe = min((eng.probe_potrf(big, alone=alone) for _ in range(3)), key=lambda r: r["total_ms"])
    syrk_tflops = probe["syrk_flops"] / (probe["syrk_ms"] / 1e3) / 1e12 if probe["syrk_ms"] > 0 else 0.0
    # a lone system with mp < 8192 is factorised by the dataflow kernel (csrc/potrf_df.cuh):
    # that one launch is the dominant kernel (no separate SYRK launches to time)
    dataflow = alone and nb_big < 64 and not ozaki and os.environ.get("PKRR_DF", "1") != "0"
    df_tflops = probe["chol_flops"] / (probe["total_ms"] / 1e3) / 1e12 if probe["total_ms"] > 0 else 0.0

    # --- e2e: public API with pinned HOST buffers (H2D + D2H inside the region) ---
    h = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in dd.items()}
    e2e_ms = []
    with torch.cuda.stream(stream):
        step(h)  # untimed: the first host-input call allocates the engine's input staging buffers
        torch.cuda.synchronize()
        for i in range(max(1, min(args.steps, 3))):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step(h)
            b.record(stream)
            b.synchronize()
            e2e_ms.append(a.elapsed_time(b))
    e2e = statistics.mean(e2e_ms)
    if world > 1:
        tt = torch.tensor([e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = float(tt.item())
    h2d = sum(v.nbytes for v in dd.values())
    d2h = ncell * (8 * 4 + 1) + 8 * (cfg["val"] + cfg["test"]) + ncell * p * (8 * 3 + 1) + 8 * 3 * p

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if cfg["scale_n"] else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (datagen.py seed 1, BASELINE {cfg['name'].split(':')[0]} shapes)",
        "config": {"workload": f"BASELINE {cfg['name']}", "strategy": cfg["strategy"],
                   "trailing_update": ("int8 Ozaki emulation of FP64 (tcgen05 kind::i8, opt-in)"
                                       if os.environ.get("PKRR_SYRK") == "ozaki" else "FP64 DMMA tensor cores"),
                   "n_train": n_train, "n_val": cfg["val"], "n_test": cfg["test"], "d": cfg["d"], "p": p,
                   "sigmas": cfg["sigmas"], "lambdas": cfg["lambdas"], "cells": ncell,
                   "samples_per_step": samples,
                   "parallelism": f"parts sharded over {world} rank(s), LPT on m^3"
                                  + (", partition sharded (NCCL all-gather per Lloyd iteration)" if shard else ""),
                   "l2": "256 MB buffer written between timed steps (per-step K/A working set >> L2)",
                   "part_sizes": [int(x) for x in res.parts["part_sizes"]]},
        "gpu_launches": int(launches),
        "fp64_tflops_step": step_tflops,
        "phase_ms_per_step": {k: v / args.steps for k, v in phase.items()},
        "part_chol_end_ms": t.get("part_chol_end_ms"),
        "roofline": DF_ROOFLINE(big, df_tflops, peak, probe) if dataflow else {"bound": "tensor",
                     "kernel": f"dsyrk_persistent_kernel (Cholesky trailing update, DMMA f64, K={syrk_k})"
                               + (" + next-column dgemm_tn_kernel<32> (single-panel groups of a lone system)"
                                  if syrk_k == 128 else ""),
                     "achieved": syrk_tflops, "peak": peak, "unit": "TFLOP/s",
                     "frac": syrk_tflops / peak if peak else None,
                     "traffic": (SYRK_NCU_LAUNCH[syrk_k][1] + SYRK_NCU_LAUNCH[syrk_k][2]
                                 if syrk_k in SYRK_NCU_LAUNCH else None),
                     "traffic_note": syrk_traffic_note(syrk_k),
                     "peak_source": "measured live after the warm-up, best of 3: FP64 DMMA (mma.sync m8n8k4) "
                                    "probe over 148 SMs; MEASURED_PEAKS.json has no FP64 entry",
                     "algorithmic": "per launch rows(rows+1)*K flops (lower triangle incl. diagonal) / launch time; "
                                    f"standalone factorization of the largest part (m={big}), "
                                    f"{probe['syrk_launches']} launches, {probe['syrk_ms']:.2f} ms of "
                                    f"{probe['total_ms']:.2f} ms"},
        "cholesky_phase": {"achieved": chol_tflops, "peak": peak, "unit": "TFLOP/s",
                           "frac": chol_tflops / peak if peak else None,
                           "algorithmic": "sum over parts and cells of m(m+1)(2m+1)/6 (solver.cpp:39-42) / union "
                                          "of the per-part Cholesky intervals in the timed steps",
                           "largest_part_alone_tflops": probe["chol_flops"] / (probe["total_ms"] / 1e3) / 1e12},
        "mse": {"selection_best": float(sel_mse[best]) if best >= 0 else None,
                "eval_of_best": float(eval_mse[best]) if best >= 0 else None, "best_index": int(best)},
        "e2e": {"value": samples / (e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e},
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        n_s = sample_rows(cfg, args.steps, args.warmup, args.sample_n)
        try:
            r, dt, (Xs, ys, Xq, yq) = reference_sample(cfg, dd, n_s, cores)
            cpu_v = (n_s + cfg["val"] + cfg["test"]) * ncell / dt
            # the same sample through the GPU engine: MSE match against the reference
            gs = eng.grid_search(cfg["strategy"], Xs, ys, Xq, yq, cfg["p"], cfg["lambdas"], cfg["sigmas"], 1)
            ok = ~r["failed"]
            rel = float(np.max(np.abs(gs.mse[ok] - r["mse"][ok]) / np.abs(r["mse"][ok]))) if ok.any() else None
            line["cpu_baseline"] = {
                "value": cpu_v, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"first {n_s} train rows, {cfg['strategy']} p={cfg['p']}, {ncell} cell(s), "
                          f"{cfg['val'] + cfg['test']} val+test rows, reference grid_search workers={cores}, "
                          f"{dt:.2f} s",
                "extrapolated_full_value": cpu_v * (cfg["n"] + cfg["val"] + cfg["test"])
                / (n_s + cfg["val"] + cfg["test"]) / cpu_extrapolation(cfg, dd, n_s, cores)[0],
                "mse_reference": [float(x) for x in r["mse"]], "mse_gpu_same_sample": [float(x) for x in gs.mse],
                "mse_max_rel_diff": rel, "best_cell_equal": bool(gs.best_index == r["best"])}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
        try:
            line["cpu_baseline"]["full_size_parity"] = full_size_parity(args.config, eng, dd)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"]["full_size_parity"] = {"unavailable": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()
    return 0


def visible_gpus():
    fake = os.environ.get("PKRR_BENCH_FAKE_GPUS")  # CPU tests of the launcher only
    if fake is not None:
        return int(fake)
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: N ranks, one per GPU, under
    torch.distributed.run (the driver's own launch shape).  Fails loudly when fewer
    than N GPUs are visible."""
    have = visible_gpus()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=dict(os.environ, PKRR_BENCH_LAUNCHED="1"))


def main():
    args = parse()
    if args.config is None:
        args.config = "c1" if args.gpus <= 1 else "c3"
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        return relaunch(args)
    if world and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if os.environ.get("PKRR_BENCH_DRYRUN"):  # launcher test: report the rank layout only
        rank, world, local = dist_env()
        # one write(2) per line: the ranks share the launcher's stdout pipe
        os.write(1, (json.dumps({"rank": rank, "world": world, "local_rank": local, "config": args.config}) + "\n").encode())
        return 0
    if args.update == "int8":  # read by the library at context creation
        os.environ["PKRR_SYRK"] = "ozaki"
    if args.impl == "reference":
        return run_reference(args)
    if visible_gpus() < max(1, world):
        print(f"bench.py: needs {max(1, world)} visible GPU(s), found {visible_gpus()}", file=sys.stderr)
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
