"""Franka cube-stack env (BSIM_TASK_STACK, BASELINE.json config 4).

The reference has this task's reward (franka_stack_reward,
rewards.py:200-219) but no env: the fused task tail is checked against a
torch restatement of the documented obs layout (include/batchsim_b200.h,
BSIM_TASK_STACK) and against the device reward kernel (pinned to the
reference by the `rewards` golden fixture): obs after every step, reward of
every env that did not reset, done = stacked | timeout, reset rows,
partition independence and the host-buffer step.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _make(**kw):
    from paper_2108_10470_b200.envs import make_env
    kw.setdefault("num_envs", 32)
    kw.setdefault("seed", 5)
    return make_env("franka-cube-stack", **kw)


def _rows(env):
    s = env.scene
    E, B = env.config.num_envs, s.bodies_per_env
    return s.body_q.view(E, B, 13).double()


def _restated_obs(env):
    s = env.scene
    E, D, B = env.config.num_envs, s.dofs_per_env, s.bodies_per_env
    dof = s.dof_state.view(E, D, 2).double()
    lo, hi = env.dof_lower.double(), env.dof_upper.double()
    r = _rows(env)
    h, a, b = r[:, B - 5], r[:, B - 2], r[:, B - 1]
    return torch.cat([2 * (dof[..., 0] - lo) / (hi - lo) - 1, 0.1 * dof[..., 1], h[:, 0:7], a[:, 0:7],
                      a[:, 0:3] - h[:, 0:3], b[:, 0:7], a[:, 0:3] - b[:, 0:3], env.actions.double()], 1)


def _stacked(env):
    from paper_2108_10470_b200 import rewards as RW
    p = RW.FrankaStackParams()
    r = _rows(env)
    B = r.shape[1]
    a, b, g = r[:, B - 2, 0:3], r[:, B - 1, 0:3], r[:, B - 5, 0:3]
    xy = (a[:, 0:2] - b[:, 0:2]).norm(dim=1)
    return (a[:, 2] > b[:, 2]) & (xy < p.align_tolerance) & ((g - a).norm(dim=1) > p.away_distance)


def _check_reset_rows(env, rows):
    from paper_2108_10470_b200 import models as M
    if rows.numel() == 0:
        return
    s = env.scene
    E, D, B = env.config.num_envs, s.dofs_per_env, s.bodies_per_env
    r = _rows(env)[rows]
    for body, spawn in ((B - 2, M.FRANKA_CUBE_A_SPAWN), (B - 1, M.FRANKA_CUBE_B_SPAWN)):
        c = r[:, body]
        sp = torch.tensor(spawn, dtype=torch.float64, device=c.device)
        assert float((c[:, 0:2] - sp[0:2]).abs().max()) <= 0.05 + 1e-6
        assert torch.allclose(c[:, 2], sp[2].expand_as(c[:, 2]), atol=1e-6)
        assert float(c[:, 3:5].abs().max()) <= 1e-6 and float(c[:, 7:13].abs().max()) == 0.0
    q = s.dof_state.view(E, D, 2)[rows].double()
    assert float(q[..., 0].abs().max()) <= 0.1 + 1e-6 and float(q[..., 1].abs().max()) == 0.0
    assert int(env.episode_steps[rows].abs().max()) == 0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_stack_task_tail_matches_restatement(precision):
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200 import rewards as RW
    env = _make(precision=precision, episode_length=30)
    E, B = env.config.num_envs, env.scene.bodies_per_env
    tol = 1e-9 if precision == "fp64" else 2e-4
    assert torch.allclose(env.obs.double(), _restated_obs(env), atol=tol, rtol=tol)
    _check_reset_rows(env, torch.arange(E, device=env.obs.device))
    g = torch.Generator(device=env.obs.device).manual_seed(5)
    ep = torch.zeros(E, dtype=torch.int64, device=env.obs.device)
    for t in range(35):
        if t == 6:   # stack cube A on cube B in envs 0..3 (gripper far above): done next step
            bq = env.scene.body_q.view(E, B, 13)
            bq[0:4, B - 2, 0:7] = bq[0:4, B - 1, 0:7]
            bq[0:4, B - 2, 2] += M.CUBE_A_HALF + M.CUBE_B_HALF + 0.0005
            bq[0:4, B - 2, 7:13] = 0
        a = torch.rand((E, env.act_dim), generator=g, device=env.obs.device, dtype=env.scene.dtype) * 2.4 - 1.2
        obs, rew, done, info = env.step(a)
        assert torch.allclose(obs.double(), _restated_obs(env), atol=tol, rtol=tol), t
        keep = ~done
        r = _rows(env)
        want = RW.franka_stack_reward(r[:, B - 2, 0:3], r[:, B - 1, 0:3], r[:, B - 5, 0:3], r[:, B - 4, 0:3],
                                      r[:, B - 3, 0:3], RW.FrankaStackParams())
        rt = 1e-9 if precision == "fp64" else 1e-4
        assert torch.allclose(rew.double()[keep], want[keep], atol=rt, rtol=rt), t
        assert not bool((keep & _stacked(env)).any())
        if t == 6:
            assert bool(done[0:4].all()) and bool((rew[0:4] == 16.0).all())
        ep += 1
        assert torch.equal(info["timeout"], ep >= 30), t
        ep[done] = 0
        _check_reset_rows(env, done.nonzero().flatten())
        assert bool(torch.isfinite(obs).all())
    env.close()


def test_stack_env_partition_independent_and_host_step():
    whole = _make(precision="fp64", num_envs=16, seed=13, episode_length=5)
    shard = _make(precision="fp64", num_envs=8, seed=13, episode_length=5, env_offset=8, total_envs=16)
    host = _make(precision="fp64", num_envs=16, seed=13, episode_length=5)
    rng = np.random.default_rng(1)
    for _ in range(7):
        a = rng.uniform(-1, 1, (16, whole.act_dim))
        ow = whole.step(torch.as_tensor(a, device=whole.obs.device))
        os_ = shard.step(torch.as_tensor(a[8:], device=whole.obs.device))
        oh = host.step_host(torch.as_tensor(a).pin_memory())
        assert torch.allclose(ow.obs[8:], os_.obs, atol=1e-12, rtol=0)
        assert torch.equal(ow.done[8:], os_.done)
        assert torch.allclose(ow.obs.cpu(), oh.obs, atol=1e-12, rtol=0)
        assert torch.equal(ow.done.cpu(), oh.done) and torch.allclose(ow.reward.cpu(), oh.reward, atol=1e-12)
    for e in (whole, shard, host):
        e.close()


def test_stack_env_long_rollout_with_graph():
    env = _make(precision="fp32", num_envs=256, randomize=True)
    env.capture_graph()
    g = torch.Generator(device=env.obs.device).manual_seed(2)
    for _ in range(120):
        obs, rew, done, info = env.step(torch.rand((256, env.act_dim), generator=g, device=env.obs.device) * 2 - 1)
    assert bool(torch.isfinite(obs).all()) and bool(torch.isfinite(rew).all())
    assert not bool(info["poisoned"].any())
    env.close()
