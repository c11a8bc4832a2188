"""bench.py's multi-GPU plumbing on CPU (no GPU work): `--gpus 2` without a
torchrun environment spawns two ranks, they rendezvous on 127.0.0.1 over
gloo, the per-rank time is reduced with MAX, and rank 0 alone prints one
JSON line with n_gpus = 2 and both ranks' records; a --gpus / WORLD_SIZE
mismatch is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None, timeout=180):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, timeout=timeout, env=e, cwd=ROOT)


def test_bench_gpus2_spawns_two_ranks():
    r = run(["--gpus", "2", "--launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["comm"]["world_size"] == 2
    assert sorted(x["rank"] for x in d["ranks"]) == [0, 1]
    assert len({x["pid"] for x in d["ranks"]}) == 2
    assert abs(d["max_rank_ms"] - 2.0) < 1e-9          # max over ranks, not rank 0's own 1.0


def test_bench_single_rank_default():
    r = run(["--launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["n_gpus"] == 1


def test_bench_gpus_world_mismatch_refused():
    r = run(["--gpus", "2", "--launch-check"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in r.stderr
