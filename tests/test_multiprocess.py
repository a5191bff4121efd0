"""Multi-process sharding on CPU (gloo, world_size 2): the host logic of the
multi-GPU path.

Each rank owns `shard_range(total, 2, rank)` of a global env batch, builds
its env origins on the global grid and keys per-env randomness on the
global env id, steps its shard (with the float64 C oracle -- the physics is
per-env and the oracle is the CPU stand-in here), and the gathered result must
be bitwise identical to one process stepping every env: the reference's
partition-independence contract (tests/test_parallel.py:37-52)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

E, STEPS = 6, 25


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_shard(lo, hi, total):
    from oracle.oracle import OracleScene
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.layout import SceneLayout
    from paper_2108_10470_b200.params import SimParams
    origins = SceneLayout([M.quadruped()]).default_env_origins(total)[lo:hi]
    s = OracleScene([M.quadruped()], hi - lo, SimParams(dt=1 / 120), env_origins=origins)
    B, D = s.bodies_per_env, s.dofs_per_env
    for k, e in enumerate(range(lo, hi)):      # per-env perturbation keyed on the GLOBAL id
        r = np.random.default_rng([9, e])
        s.pos[k * B:(k + 1) * B, 2] += 0.37
        s.gravity[k, 2] = -9.81 * r.uniform(0.8, 1.2)
        s.mu_static[k] = s.mu_dynamic[k] = r.uniform(0.5, 1.5)
    s.forward_kinematics()
    for t in range(STEPS):
        for k, e in enumerate(range(lo, hi)):
            s.ctrl_dof_pos_target[k * D:(k + 1) * D] = np.random.default_rng([9, e, t]).uniform(-0.5, 0.5, D)
        s.step()
    return np.concatenate([s.pos, s.quat, s.linvel, s.angvel], 1), s.dof_state.copy()


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2108_10470_b200.parallel import rollout_stats, shard_range
    lo, hi = shard_range(E, world, rank)
    body, dof = _run_shard(lo, hi, E)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, body, dof))
    stats = rollout_stats(torch.full((hi - lo,), float(rank + 1)), torch.ones(hi - lo, dtype=torch.bool))
    if rank == 0:
        np.savez(out_path, body=np.concatenate([g[2] for g in sorted(gathered, key=lambda g: g[0])]),
                 dof=np.concatenate([g[3] for g in sorted(gathered, key=lambda g: g[0])]),
                 stats=np.array(stats, dtype=np.float64))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_step_partition_independent_gloo(tmp_path, world):
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    z = np.load(out)
    body, dof = _run_shard(0, E, E)
    assert np.array_equal(z["body"], body)
    assert np.array_equal(z["dof"], dof)
    # rollout_stats: mean reward over all ranks' envs, finished episodes, env count
    from paper_2108_10470_b200.parallel import shard_bounds
    b = shard_bounds(E, world)
    want = sum((r + 1) * (b[r + 1] - b[r]) for r in range(world)) / E
    assert z["stats"][0] == pytest.approx(want) and z["stats"][1] == E and z["stats"][2] == E


def test_shard_bounds_match_reference_partition():
    from paper_2108_10470_b200.parallel import shard_bounds, shard_range
    for total, world in ((16384, 8), (6, 5), (7, 3)):
        b = shard_bounds(total, world)
        assert b[0] == 0 and b[-1] == total and np.all(np.diff(b) >= 0)
        assert np.array_equal(b, np.linspace(0, total, world + 1).astype(int))   # parallel.py:102
        assert sum(hi - lo for lo, hi in (shard_range(total, world, r) for r in range(world))) == total
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
