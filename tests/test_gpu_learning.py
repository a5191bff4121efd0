"""Acceptance: PPO on the GPU env batch learns to walk forward.

Mirrors the reference's `test_accept_quadruped_learning`
(tests/test_acceptance.py:222-288): 128 envs, horizon 16, 150 PPO
iterations, progress = mean forward speed (local root x rate) of the envs
still alive after each control step, averaged over the last 100 iterations;
at least 2 of 3 seeds must make positive progress.  Here the env runs in the
CUDA step kernel and the policy / update in PyTorch on the same device.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _quadruped_progress(seed, iters=150, num_envs=128, horizon=16):
    from paper_2108_10470_b200.envs import make_env
    from paper_2108_10470_b200.ppo import PPO, gae_advantages
    env = make_env("quadruped", num_envs=num_envs, seed=seed)
    dev = env.obs.device
    agent = PPO(env.obs_dim, env.act_dim, seed=seed, device=dev)
    obs = env.reset().clone()
    dt = env.config.control_dt
    hist = []
    for _ in range(iters):
        T, E = horizon, num_envs
        O = torch.empty((T, E, env.obs_dim), device=dev)
        A = torch.empty((T, E, env.act_dim), device=dev)
        LP, V, R, D = (torch.empty((T, E), device=dev) for _ in range(4))
        prog = []
        with torch.no_grad():
            for t in range(T):
                a, lp, v = agent.net.act(obs, agent.gen)
                O[t], A[t], LP[t], V[t] = obs, a, lp, v
                x0 = env.local_root()[:, 0].clone()
                out = env.step(a)
                alive = ~out.done
                if bool(alive.any()):
                    x1 = env.local_root()[:, 0]
                    prog.append(float(((x1[alive] - x0[alive]) / dt).mean()))
                obs = out.obs.clone()
                R[t], D[t] = out.reward, out.done.float()
            last = agent.net.value(obs)
        adv, ret = gae_advantages(R, V, D, last, 0.99, 0.95)
        flat = lambda x: x.reshape(-1, *x.shape[2:])  # noqa: E731
        agent.update(flat(O), flat(A), LP.reshape(-1), V.reshape(-1), adv.reshape(-1), ret.reshape(-1))
        hist.append(sum(prog) / max(1, len(prog)))
    env.close()
    return sum(hist[-100:]) / 100.0


def test_quadruped_learns_forward_progress():
    progress = [_quadruped_progress(seed) for seed in (0, 1, 2)]
    wins = sum(p > 0.0 for p in progress)
    assert wins >= 2, progress


def test_throughput_scales_with_envs():
    """Reference test_accept_throughput_scaling (tests/test_acceptance.py:
    168-219) on the device: 16384 envs step >= 4x the env-steps/s of 1024
    envs (the batch fills the 148 SMs instead of a fraction of one wave)."""
    from paper_2108_10470_b200.envs import make_env

    def fps(E, steps=20):
        env = make_env("quadruped", num_envs=E, seed=0)
        a = torch.rand((E, env.act_dim), device=env.obs.device) * 2 - 1
        for _ in range(3):
            env.step(a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            env.step(a)
        e1.record()
        torch.cuda.synchronize()
        env.close()
        return E * steps / (e0.elapsed_time(e1) / 1e3)

    ratio = fps(16384) / fps(1024)
    assert ratio >= 4.0, ratio
