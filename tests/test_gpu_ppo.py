"""PPO caller + CLI on the GPU env batch (float32 policy in PyTorch, envs in
the CUDA step kernel).  Single GPU; the NCCL paths are covered by the gloo
world-size-2 tests in tests/test_ppo.py and the torchrun launch in bench.py."""

import csv

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_train_two_iterations_on_quadruped(tmp_path):
    from paper_2108_10470_b200 import cli
    rc = cli.main(["train", "--env", "quadruped", "--num-envs", "256", "--iterations", "2", "--horizon", "8",
                   "--out", str(tmp_path)])
    assert rc == 0
    rows = list(csv.DictReader(open(tmp_path / "metrics.csv")))
    assert [int(r["env_steps"]) for r in rows] == [2048, 4096]
    assert all(float(r["loss"]) == float(r["loss"]) for r in rows)          # finite
    assert (tmp_path / "checkpoint.bin").stat().st_size > 40
    rc = cli.main(["eval", "--env", "quadruped", "--num-envs", "64", "--episodes", "1",
                   "--checkpoint", str(tmp_path / "checkpoint.bin")])
    assert rc == 0


def test_bench_csv(tmp_path):
    from paper_2108_10470_b200 import cli
    out = tmp_path / "bench.csv"
    rc = cli.main(["bench", "--env", "quadruped-anymal-obs", "--num-envs", "256,1024", "--base-horizon", "8",
                   "--warmup", "3", "--out", str(out)])
    assert rc == 0
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0]) == ["num_envs", "horizon", "control_steps_per_sec", "sim_steps_per_sec", "wall_clock_s"]
    assert [int(r["horizon"]) for r in rows] == [8, 2]
    for r in rows:
        assert float(r["sim_steps_per_sec"]) == pytest.approx(2 * float(r["control_steps_per_sec"]))


def test_collect_rollout_shapes():
    from paper_2108_10470_b200.envs import make_env
    from paper_2108_10470_b200.ppo import PPO, PPOConfig, collect_rollout, gae_advantages
    env = make_env("quadruped", num_envs=128, seed=3)
    agent = PPO(env.obs_dim, env.act_dim, PPOConfig(hidden=(64, 64)), device=env.scene.device)
    roll, obs = collect_rollout(env, agent, env.reset(), 6)
    assert roll["obs"].shape == (6, 128, 60) and roll["actions"].shape == (6, 128, 8)
    assert torch.isfinite(roll["rewards"]).all() and torch.isfinite(roll["values"]).all()
    adv, ret = gae_advantages(roll["rewards"], roll["values"], roll["dones"], roll["last_value"], 0.99, 0.95)
    assert adv.shape == (6, 128) and torch.isfinite(ret).all()
    env.close()


def test_policy_graph_matches_eager_act():
    """ppo.PolicyGraph (act() as one CUDA graph) returns what act() returns:
    the value and log-probability of its own sample exactly as the eager
    functions compute them, the sample's noise with the policy's std, and a
    generator stream that continues across replays (no repeated noise)."""
    import torch
    from paper_2108_10470_b200.ppo import PPO, PolicyGraph
    agent = PPO(60, 8, device="cuda")
    obs = torch.randn(4096, 60, device="cuda")
    pg = PolicyGraph(agent.net, agent.gen, obs)
    a1, lp1, v1 = (x.clone() for x in pg(obs))
    a2, _, _ = (x.clone() for x in pg(obs))
    net = agent.net
    with torch.no_grad():
        mu = net.actor(obs)
        assert torch.allclose(v1, net.value(obs), atol=1e-6)
        assert torch.allclose(lp1, net._log_prob(mu, a1, net._log_std_c()), atol=1e-4)
        z = (a1 - mu) / torch.exp(net._log_std_c())
    assert abs(float(z.mean())) < 0.02 and abs(float(z.std()) - 1.0) < 0.02
    assert not torch.equal(a1, a2)                     # the stream moved on between replays
