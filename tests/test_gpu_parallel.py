"""Partition independence of the GPU path (reference tests/test_parallel.py:37-52):
shards built with global env offsets reproduce the single-scene run bitwise."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _perturb_and_run(s, lo, steps=30):
    B, D = s.bodies_per_env, s.dofs_per_env
    s.pos[:, 2] += 0.37
    for k in range(s.num_envs):
        r = np.random.default_rng([9, lo + k])
        s.gravity[k, 2] = -9.81 * r.uniform(0.8, 1.2)
    s.forward_kinematics()
    for t in range(steps):
        tgt = np.concatenate([np.random.default_rng([9, lo + k, t]).uniform(-0.5, 0.5, D)
                              for k in range(s.num_envs)])
        s.ctrl_dof_pos_target.copy_(torch.as_tensor(tgt, dtype=s.dtype))
        s.step(2)
    return s.body_q.cpu().numpy(), s.root_state.cpu().numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_scene_shards_bitwise_equal_to_full(world):
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.parallel import shard_range
    from paper_2108_10470_b200.scene import Scene
    E = 48
    full = _perturb_and_run(Scene([M.quadruped()], E), 0)
    parts = []
    for r in range(world):
        lo, hi = shard_range(E, world, r)
        parts.append(_perturb_and_run(Scene([M.quadruped()], hi - lo, env_offset=lo, total_envs=E), lo))
    assert np.array_equal(np.concatenate([p[0] for p in parts]), full[0])
    assert np.array_equal(np.concatenate([p[1] for p in parts]), full[1])   # world-frame origins too


def test_sharded_env_resets_use_global_ids():
    from paper_2108_10470_b200.parallel import make_sharded_env
    from paper_2108_10470_b200.envs import make_env
    full = make_env("quadruped", num_envs=10, seed=3)
    a = make_sharded_env("quadruped", 10, rank=0, world=2, seed=3)
    b = make_sharded_env("quadruped", 10, rank=1, world=2, seed=3)
    assert torch.equal(torch.cat([a.obs, b.obs]), full.obs)
    assert torch.equal(torch.cat([a.scene.root_state, b.scene.root_state]), full.scene.root_state)
