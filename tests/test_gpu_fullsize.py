"""Size-independent properties at the benchmark's full size (BASELINE.json:
16384 envs per GPU): the per-env result does not depend on how envs are
packed into CTAs (whole-wave balancing changes the envs per CTA with the
batch size; the large-articulation variant uses 4-env CTAs), long rollouts
stay finite, and the fp32 step stays within the parity contract of the
float64 oracle at 16384 envs."""

import os

import numpy as np
import pytest
import torch

from golden_util import rel_err

pytestmark = pytest.mark.gpu

E_FULL = 16384


def _walkers(model_name, E, seed=0, precision="fp32"):
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.layout import SceneLayout
    from paper_2108_10470_b200.params import SimParams
    from paper_2108_10470_b200.scene import Scene
    model = getattr(M, model_name)()
    origins = SceneLayout([model]).default_env_origins(E_FULL)[:E]
    s = Scene([model], E, SimParams(dt=1 / 120), env_origins=origins, precision=precision)
    rest = {"quadruped": M.QUADRUPED_REST_HEIGHT, "quadruped12": M.QUADRUPED12_REST_HEIGHT,
            "humanoid": M.HUMANOID_REST_HEIGHT}[model_name]
    s.pos[:, 2] += rest + 0.02
    g = np.random.default_rng(seed)
    dof = torch.as_tensor(g.uniform(-0.1, 0.1, (E_FULL, s.dofs_per_env))[:E].reshape(-1), dtype=s.dtype)
    s.dof_state[:, 0] = dof.to(s.device)
    s.forward_kinematics()
    return s


@pytest.mark.parametrize("model_name", ["quadruped", "quadruped12", "humanoid"])
def test_results_independent_of_cta_packing(model_name):
    """16384 envs in one scene == the first 1000 of them in a 1000-env scene
    (different envs per CTA, different grid), bitwise, over 6 control steps."""
    big = _walkers(model_name, E_FULL)
    small = _walkers(model_name, 1000)
    g = np.random.default_rng(7)
    D = big.dofs_per_env
    for _ in range(6):
        a = torch.as_tensor(g.uniform(-1, 1, (E_FULL, D)), dtype=torch.float32, device="cuda")
        big.step(2, actions=a, action_scale=0.6)
        small.step(2, actions=a[:1000].contiguous(), action_scale=0.6)
    B = big.bodies_per_env
    assert torch.equal(big.body_q[: 1000 * B], small.body_q)
    assert torch.equal(big.dof_state[: 1000 * D], small.dof_state)
    assert torch.equal(big.net_contact[: 1000 * B], small.net_contact)


@pytest.mark.parametrize("task", ["quadruped", "humanoid"])
def test_long_rollout_stays_finite(task):
    """300 control steps of random actions at 16384 envs through EnvBatch
    (auto-resets included): no env is poisoned, obs / reward stay finite."""
    from paper_2108_10470_b200.envs import make_env
    env = make_env(task, num_envs=E_FULL, seed=1)
    gen = torch.Generator(device="cuda").manual_seed(0)
    resets = 0
    for _ in range(300):
        out = env.step(torch.rand((E_FULL, env.act_dim), generator=gen, device="cuda") * 2 - 1)
        resets += int(out.done.sum())
    assert int(out.info["poisoned"].sum()) == 0 and int(env.scene.nonfinite.sum()) == 0
    assert bool(torch.isfinite(out.obs).all()) and bool(torch.isfinite(out.reward).all())
    assert resets > 0
    env.close()


def test_fp32_step_matches_oracle_at_16384_envs():
    """One teacher-forced sim step of 16384 Ant-analog envs (after 20 warm-up
    steps of the oracle) vs the float64 oracle, fp32 contract."""
    from oracle.oracle import OracleScene
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.params import SimParams
    from paper_2108_10470_b200.scene import Scene
    from golden_util import gpu_outputs
    p = SimParams(dt=1 / 120)
    ref = OracleScene([M.quadruped()], E_FULL, p, threads=os.cpu_count() or 1)
    ref.pos[:, 2] += 0.37
    ref.forward_kinematics()
    rng = np.random.default_rng(3)
    for _ in range(20):
        ref.ctrl_dof_pos_target[:] = rng.uniform(-0.6, 0.6, ref.num_dofs)
        ref.step()
    gpu = Scene([M.quadruped()], E_FULL, p)
    B = gpu.bodies_per_env
    be = np.repeat(np.arange(E_FULL), B)
    tgt = rng.uniform(-0.6, 0.6, ref.num_dofs)
    ref.ctrl_dof_pos_target[:] = tgt
    bq = np.concatenate([ref.pos - ref.env_origins[be], ref.quat, ref.linvel, ref.angvel], 1)
    gpu.body_q.copy_(torch.as_tensor(bq, dtype=gpu.dtype))
    gpu._friction_anchor.copy_(torch.as_tensor(ref._friction_anchor - ref.env_origins[None], dtype=gpu.dtype))
    gpu.dof_state.copy_(torch.as_tensor(ref.dof_state, dtype=gpu.dtype))
    gpu.ctrl_dof_pos_target.copy_(torch.as_tensor(tgt, dtype=gpu.dtype))
    ref.step()
    gpu.step()
    got = gpu_outputs(gpu)
    for k in ("root_state", "body_state", "dof_state", "net_contact", "sensor_forces"):
        e = rel_err(got[k], getattr(ref, k), 2e-3, 2e-3)
        assert e <= 1.0, (k, e)
        within = np.abs(got[k] - getattr(ref, k)) <= 1e-4 + 1e-4 * np.abs(getattr(ref, k))
        assert within.mean() >= 0.99, (k, within.mean())
