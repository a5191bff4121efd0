"""The multi-GPU path through real ranks (reference partition independence,
tests/test_parallel.py:37-52; ShardedScene env ranges, parallel.py:102-112).

One GPU is enough to run it: the ranks are separate processes sharing cuda:0
over gloo.  A 2-rank job of the product env (fused CUDA step, task tail,
auto-resets keyed on global env ids) must equal the 1-rank job per env,
bitwise; and `bench.py --gpus 2` must launch 2 ranks itself and report the
whole job."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "workers", "multirank_env.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _job(world, task, total, steps, out):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, WORKER, task, str(total), str(steps), str(out)], env=env))
    rcs = [p.wait(timeout=600) for p in procs]
    assert rcs == [0] * world, rcs
    return np.load(out)


@pytest.mark.parametrize("task", ["quadruped", "quadruped-anymal-obs"])
def test_two_rank_job_equals_one_rank_job(task, tmp_path):
    total, steps = 96, 30
    one = _job(1, task, total, steps, tmp_path / "one.npz")
    two = _job(2, task, total, steps, tmp_path / "two.npz")
    for k in ("obs", "reward", "done", "root"):
        assert np.array_equal(one[k], two[k]), k
    assert one["done"].any()                      # terminations / timeouts and auto-resets happened
    assert float(one["mean_reward"]) == float(two["mean_reward"]) and int(one["n"]) == total


def test_bench_launches_ranks_itself():
    """`python bench.py --gpus 2` outside torchrun: two ranks, whole-job value."""
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--envs", "2048", "--no-other-configs", "--no-cpu-baseline"],
                       capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_envs"] == 4096
    assert line["config"]["parallelism"] == "env-shard x2" and line["dist_backend"] == "gloo"
    assert line["value"] > 0 and line["e2e"]["value"] > 0
