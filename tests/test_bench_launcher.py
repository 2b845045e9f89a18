"""bench.py --gpus N outside torchrun: it re-launches itself under
torch.distributed.run with N ranks (RANK / WORLD_SIZE / LOCAL_RANK set per rank), and
refuses to run when fewer than N GPUs are visible (CPU test of the launcher only:
PKRR_BENCH_FAKE_GPUS stands in for the device count, PKRR_BENCH_DRYRUN stops each rank
after reporting its layout)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, **env):
    e = dict(os.environ, **env)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "PKRR_BENCH_LAUNCHED"):
        e.pop(k, None)
    e.update(env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=e, capture_output=True,
                          text=True, timeout=300)


def test_gpus_2_spawns_two_ranks():
    r = _bench(["--gpus", "2", "--steps", "1", "--warmup", "3"], PKRR_BENCH_FAKE_GPUS="2", PKRR_BENCH_DRYRUN="1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 for x in lines)
    assert sorted(x["local_rank"] for x in lines) == [0, 1]
    assert all(x["config"] == "c3" for x in lines)  # the weak-scaling config at N > 1


def test_gpus_1_is_c1_in_process():
    r = _bench(["--gpus", "1"], PKRR_BENCH_FAKE_GPUS="1", PKRR_BENCH_DRYRUN="1")
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert line == {"rank": 0, "world": 1, "local_rank": 0, "config": "c1"}


def test_gpus_2_on_one_gpu_fails_loudly():
    r = _bench(["--gpus", "2"], PKRR_BENCH_FAKE_GPUS="1")
    assert r.returncode != 0
    assert "needs 2 visible GPUs" in r.stderr


def test_no_gpu_fails_loudly():
    r = _bench(["--steps", "1"], PKRR_BENCH_FAKE_GPUS="0")
    assert r.returncode != 0
    assert "visible GPU" in r.stderr
