"""Shadow-Hand cube reorientation env (BSIM_TASK_CUBE, BASELINE.json config 5).

The reference has this task's reward (cube_reorientation_reward,
rewards.py:161-176) but no env, so the fused task tail is checked against a
torch restatement of the documented layout (include/batchsim_b200.h,
BSIM_TASK_CUBE) and against the device reward kernel, which the `rewards`
golden fixture pins to the reference: obs of every env after every step,
reward of every env that did not reset, done = fall | timeout, goal resets
on success, reset rows, partition independence and the host-buffer step.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _make(**kw):
    from paper_2108_10470_b200.envs import make_env
    kw.setdefault("num_envs", 32)
    kw.setdefault("seed", 3)
    return make_env("shadow-hand", **kw)


def _qmul(a, b):
    ax, ay, az, aw = a.unbind(-1)
    bx, by, bz, bw = b.unbind(-1)
    return torch.stack([aw * bx + ax * bw + ay * bz - az * by, aw * by - ax * bz + ay * bw + az * bx,
                        aw * bz + ax * by - ay * bx + az * bw, aw * bw - ax * bx - ay * by - az * bz], -1)


def _conj(q):
    return torch.cat([-q[..., :3], q[..., 3:]], -1)


def _cube(env):
    s = env.scene
    E, B = env.config.num_envs, s.bodies_per_env
    return s.body_q.view(E, B, 13)[:, B - 1].double()


def _restated_obs(env):
    s = env.scene
    E, D = env.config.num_envs, s.dofs_per_env
    dof = s.dof_state.view(E, D, 2).double()
    lo, hi = env.dof_lower.double(), env.dof_upper.double()
    cb, g = _cube(env), env.goals.double()
    return torch.cat([2 * (dof[..., 0] - lo) / (hi - lo) - 1, 0.2 * dof[..., 1], cb[:, 0:10], 0.2 * cb[:, 10:13],
                      g[:, 0:7], _qmul(cb[:, 3:7], _conj(g[:, 3:7])), env.actions.double()], 1)


def _check_reset_rows(env, rows):
    from paper_2108_10470_b200 import models as M
    if rows.numel() == 0:
        return
    s = env.scene
    E, D = env.config.num_envs, s.dofs_per_env
    cb = _cube(env)[rows]
    spawn = torch.tensor(M.SHADOW_CUBE_SPAWN, dtype=torch.float64, device=cb.device)
    tol = 1e-6 if s.fp64 else 1e-5
    assert torch.allclose(cb[:, 0:3], spawn.expand_as(cb[:, 0:3]), atol=tol, rtol=0)
    assert torch.allclose(cb[:, 3:5], torch.zeros_like(cb[:, 3:5]), atol=tol)       # pure yaw
    assert float(cb[:, 7:13].abs().max()) == 0.0
    q = s.dof_state.view(E, D, 2)[rows].double()
    assert float(q[..., 0].abs().max()) <= 0.1 + 1e-6 and float(q[..., 1].abs().max()) == 0.0
    g = env.goals.double()[rows]
    assert torch.allclose(g[:, 3:7].norm(dim=1), torch.ones(len(rows), dtype=torch.float64, device=g.device),
                          atol=tol)
    assert float(g[:, 7].abs().max()) == 0.0
    assert int(env.episode_steps[rows].abs().max()) == 0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_cube_task_tail_matches_restatement(precision):
    from paper_2108_10470_b200 import rewards as RW
    env = _make(precision=precision, episode_length=40)
    E = env.config.num_envs
    tol = 1e-9 if precision == "fp64" else 2e-4
    assert torch.allclose(env.obs.double(), _restated_obs(env), atol=tol, rtol=tol)
    _check_reset_rows(env, torch.arange(E, device=env.obs.device))
    g = torch.Generator(device=env.obs.device).manual_seed(5)
    saw_done = False
    ep = torch.zeros(E, dtype=torch.int64, device=env.obs.device)
    for t in range(45):
        if t == 10:   # drop the cube of a few envs below the palm: they fall out of reach
            E_, B = E, env.scene.bodies_per_env
            env.scene.body_q.view(E_, B, 13)[0:4, B - 1, 2] = 0.1
        goals0 = env.goals.clone()
        a = torch.rand((E, env.act_dim), generator=g, device=env.obs.device, dtype=env.scene.dtype) * 2.4 - 1.2
        obs, rew, done, info = env.step(a)
        assert torch.allclose(obs.double(), _restated_obs(env), atol=tol, rtol=tol), t
        keep = ~done
        cb = _cube(env)
        want, _, succ = RW.cube_reorientation_reward(cb[:, 0:3], cb[:, 3:7], goals0[:, 0:3].double(),
                                                     goals0[:, 3:7].double(), env.actions.double(),
                                                     RW.CubeRewardParams())
        rt = 1e-9 if precision == "fp64" else 1e-3
        assert torch.allclose(rew.double()[keep], want[keep], atol=rt, rtol=rt), t
        dist = (cb[:, 0:3] - goals0[:, 0:3].double()).norm(dim=1)
        assert not bool((keep & (dist >= 0.24)).any())
        if t == 10:
            assert bool(done[0:4].all()) and not bool(info["timeout"][0:4].any())
        ep += 1
        assert torch.equal(info["timeout"], ep >= 40), t
        ep[done] = 0
        saw_done |= bool(done.any())
        _check_reset_rows(env, done.nonzero().flatten())
        assert bool(torch.isfinite(obs).all())
    assert saw_done
    env.close()


def test_success_draws_a_new_goal():
    env = _make(precision="fp64", num_envs=8)
    cb = _cube(env)
    env.goals[0:4, 3:7] = cb[0:4, 3:7]            # goal = the current orientation: success next step
    flip = torch.tensor([1.0, 0.0, 0.0, 0.0], dtype=torch.float64, device=cb.device).expand(4, 4)
    env.goals[4:8, 3:7] = _qmul(cb[4:8, 3:7], flip)  # half a turn away: no success
    old = env.goals.clone()
    obs, rew, done, _ = env.step(torch.zeros((8, env.act_dim), dtype=torch.float64, device=env.obs.device))
    assert not bool(done.any())
    assert bool((rew[0:4] > 200).all()) and bool((rew[4:] < 200).all())
    assert torch.equal(env.successes[0:4], torch.ones(4, dtype=torch.float64, device=env.obs.device))
    assert float(env.successes[4:].abs().max()) == 0.0
    assert not torch.allclose(env.goals[0:4, 3:7], old[0:4, 3:7])
    assert torch.equal(env.goals[4:], old[4:])
    assert torch.allclose(env.goals[:, 3:7].norm(dim=1), torch.ones(8, dtype=torch.float64, device=env.obs.device))
    env.close()


def test_cube_env_partition_independent_and_host_step():
    """A shard (env_offset 8 of 16) reproduces rows 8..16 of the whole batch,
    and step_host (pinned host actions, pipelined chunks) equals step()."""
    whole = _make(precision="fp64", num_envs=16, seed=11, episode_length=6)
    shard = _make(precision="fp64", num_envs=8, seed=11, episode_length=6, env_offset=8, total_envs=16)
    host = _make(precision="fp64", num_envs=16, seed=11, episode_length=6)
    rng = np.random.default_rng(0)
    for _ in range(8):
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


def test_cube_env_with_domain_randomisation_and_graph():
    env = _make(precision="fp32", num_envs=64, randomize=True, obs_noise=True)
    env.capture_graph()
    g = torch.Generator(device=env.obs.device).manual_seed(1)
    for _ in range(30):
        obs, rew, done, info = env.step(torch.rand((64, env.act_dim), generator=g, device=env.obs.device) * 2 - 1)
    assert bool(torch.isfinite(obs).all()) and bool(torch.isfinite(rew).all())
    assert not bool(info["poisoned"].any())
    env.close()
