"""Random object forces on the device vs the reference's contract
(randomize.py:192-221; the reference's own tests test_randomize.py:101-132,
restated here against the device implementation)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_random_force_decay_exact(dtype):
    from paper_2108_10470_b200.randomize import RandomForceState, random_object_force
    state = RandomForceState(num_envs=1, rng=np.random.default_rng(0), dtype=dtype)
    state.probability[:] = 0.0
    state.force[:] = torch.tensor([3.0, -4.0, 0.0], dtype=dtype)
    f = random_object_force(state, mass=np.ones(1), dt=0.05).double().cpu().numpy()
    tol = 1e-12 if dtype == torch.float64 else 1e-6
    assert np.allclose(f, np.array([[3.0, -4.0, 0.0]]) * 0.99, atol=tol, rtol=tol)
    assert abs(np.linalg.norm(f) - 0.99 * 5.0) < (1e-12 if dtype == torch.float64 else 1e-5)


def test_random_force_zero_probability_stays_zero():
    from paper_2108_10470_b200.randomize import RandomForceState, random_object_force
    state = RandomForceState(num_envs=4, rng=np.random.default_rng(0))
    state.probability[:] = 0.0
    for _ in range(100):
        f = random_object_force(state, mass=np.ones(4), dt=1 / 120)
        assert bool((f == 0.0).all())


def test_random_force_refresh_std():
    from paper_2108_10470_b200.randomize import RandomForceState, random_object_force
    state = RandomForceState(num_envs=1_000_000, rng=np.random.default_rng(1), dtype=torch.float64)
    state.probability[:] = 1.0
    f = random_object_force(state, mass=np.full(1_000_000, 2.0), dt=1 / 120)
    assert abs(float(f.std()) - 2.0) / 2.0 < 0.01
    assert abs(float(f.mean())) < 5 * 2.0 / math.sqrt(f.numel())


def test_force_probability_range():
    from paper_2108_10470_b200.randomize import RandomForceState
    state = RandomForceState(num_envs=100_000, rng=np.random.default_rng(2), dtype=torch.float64)
    p = state.probability.cpu().numpy()
    assert p.min() >= 0.001 and p.max() <= 0.1
    logs = np.log(p)
    mid = (math.log(0.001) + math.log(0.1)) / 2
    assert abs(logs.mean() - mid) < 3 * logs.std() / math.sqrt(len(logs))


def test_fire_rate_and_partition_independence():
    """Fire frequency equals p; per-env streams are keyed by global env id, so
    a shard [lo, hi) reproduces the same rows of a full batch."""
    from paper_2108_10470_b200.randomize import RandomForceState, random_object_force
    E = 20000
    full = RandomForceState(E, rng=7, dtype=torch.float64)
    full.probability[:] = 0.25
    shard = RandomForceState(E // 4, rng=7, dtype=torch.float64, env_offset=E // 2)
    shard.probability[:] = 0.25
    fired = 0
    for _ in range(8):
        prev = full.force.clone()
        f = random_object_force(full, mass=np.ones(E), dt=1 / 120)
        g = random_object_force(shard, mass=np.ones(E // 4), dt=1 / 120)
        assert torch.equal(f[E // 2:E // 2 + E // 4], g)
        fired += int((f != prev * 0.99 ** ((1 / 120) / 0.05)).any(1).sum())
    rate = fired / (8 * E)
    assert abs(rate - 0.25) < 0.01
    # resample_probability redraws p and zeroes the force of the given envs only
    full.resample_probability([0, 5])
    assert float(full.force[[0, 5]].abs().sum()) == 0.0
    assert float(full.probability[1]) == 0.25
    p = full.probability[[0, 5]].cpu().numpy()
    assert (p >= 0.001).all() and (p <= 0.1).all()


def test_force_written_into_scene_controls():
    """The fused write lands in the object's ctrl_body_force row and moves it."""
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.randomize import RandomForceState, random_object_force
    from paper_2108_10470_b200.scene import Scene
    s = Scene([M.quadruped()], 8, precision="fp32")
    st = RandomForceState(8, rng=3, device=s.device)
    st.probability[:] = 1.0
    mass = 1.0 / s.inv_mass.reshape(8, -1)[:, 0]
    f = random_object_force(st, mass, dt=1 / 120, body_force=s.ctrl_body_force, body=0,
                            bodies_per_env=s.bodies_per_env)
    rows = s.ctrl_body_force.reshape(8, s.bodies_per_env, 3)
    assert torch.equal(rows[:, 0], f)
    assert float(rows[:, 1:].abs().sum()) == 0.0
    with pytest.raises(ValueError):
        random_object_force(st, np.ones(3), dt=1 / 120)
