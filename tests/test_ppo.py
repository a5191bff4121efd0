"""The PPO caller of the hot path (paper_2108_10470_b200/ppo.py) against
golden vectors produced by the reference's own ppo.py
(tests/golden/make_ppo_golden.py), plus the data-parallel contract over
gloo (world size 2): a 2-rank update on two halves of a batch equals a
1-rank update on the whole batch.  Float64 on CPU; mirrors the reference's
tests/test_ppo.py (GAE oracle, gradients, Adam, checkpoint, bandit)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_10470_b200 import ppo as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")
D64 = torch.float64


@pytest.fixture(scope="module")
def z():
    return np.load(os.path.join(GOLD, "ppo.npz"))


def _t(a):
    return torch.as_tensor(np.asarray(a), dtype=D64)


def _agent(z):
    cfg = P.PPOConfig(hidden=(32, 16), minibatch_size=64, epochs=1, entropy_coef=0.01)
    a = P.PPO(7, 3, cfg, seed=3, dtype=D64)
    n = len(a.net.params())
    a.net.set_params([z[f"param0_{i}"] for i in range(n)])
    return a


def _batch(z):
    return tuple(_t(z[k]) for k in ("obs", "act", "logp_old", "v_old", "adv", "ret"))


def test_gae_matches_reference(z):
    adv, ret = P.gae_advantages(_t(z["gae_rewards"]), _t(z["gae_values"]), _t(z["gae_dones"]),
                                _t(z["gae_last"]), 0.99, 0.95)
    np.testing.assert_allclose(adv.numpy(), z["gae_adv"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ret.numpy(), z["gae_ret"], rtol=0, atol=1e-12)


def test_gae_quadratic_oracle():
    """O(T^2) definition of GAE (reference tests/test_ppo.py:15-45)."""
    rng = np.random.default_rng(1)
    T, E, g, l = 7, 4, 0.97, 0.9
    r, v, last = rng.normal(size=(T, E)), rng.normal(size=(T, E)), rng.normal(size=E)
    d = (rng.uniform(size=(T, E)) < 0.3).astype(float)
    adv, _ = P.gae_advantages(_t(r), _t(v), _t(d), _t(last), g, l)
    for e in range(E):
        for t in range(T):
            acc, coef = 0.0, 1.0
            for k in range(t, T):
                nv = last[e] if k == T - 1 else v[k + 1, e]
                delta = r[k, e] + g * nv * (1 - d[k, e]) - v[k, e]
                acc += coef * delta
                if d[k, e]:
                    break
                coef *= g * l
            assert abs(acc - float(adv[t, e])) < 1e-10


def test_initial_params_match_reference_init(z):
    a = P.PPO(7, 3, P.PPOConfig(hidden=(32, 16)), seed=3, dtype=D64)
    ps = a.net.params()
    # the reference init stream (ppo.py:108) for the weights; log_std was perturbed in the fixture
    for i, p in enumerate(ps[:-1]):
        np.testing.assert_array_equal(p.detach().numpy(), z[f"param0_{i}"])


def test_loss_and_grads_match_reference(z):
    a = _agent(z)
    stats, grads = a.net.loss_and_grads(*_batch(z))
    want = z["stats"]
    got = [stats[k] for k in ("loss", "pg_loss", "v_loss", "entropy", "kl")]
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12)
    for i, g in enumerate(grads):
        np.testing.assert_allclose(g.numpy(), z[f"grad_{i}"], rtol=1e-8, atol=1e-12)


def test_update_matches_reference(z):
    a = _agent(z)
    st = a.update(*_batch(z))
    for i, p in enumerate(a.net.params()):
        np.testing.assert_allclose(p.detach().numpy(), z[f"param1_{i}"], rtol=1e-9, atol=1e-12)
    assert st["lr"] == pytest.approx(float(z["update_lr"][0]))


def test_adam_matches_reference(z):
    ps = [_t(z["adam_p0a"]).clone(), _t(z["adam_p0b"]).clone()]
    opt = P.Adam(ps, lr=1e-2)
    opt.step(ps, [_t(z["adam_g1a"]), _t(z["adam_g1b"])])
    opt.step(ps, [_t(z["adam_g2a"]), _t(z["adam_g2b"])])
    np.testing.assert_allclose(ps[0].numpy(), z["adam_p2a"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(ps[1].numpy(), z["adam_p2b"], rtol=0, atol=1e-14)


def test_checkpoint_interoperates_with_reference(z, tmp_path):
    """A reference-written BSCK checkpoint loads bit-exactly, and saving it
    back reproduces the reference's bytes (ppo.py:319-348)."""
    ref = os.path.join(GOLD, "ppo_ckpt.bin")
    a = P.PPO(7, 3, P.PPOConfig(hidden=(32, 16)), seed=99, dtype=D64)
    a.load(ref)
    for i, p in enumerate(a.net.params()):
        np.testing.assert_array_equal(p.detach().numpy(), z[f"param0_{i}"].astype(np.float32).astype(np.float64))
    out = tmp_path / "x.bin"
    a.save(out)
    assert out.read_bytes() == open(ref, "rb").read()
    b = P.PPO(7, 4, P.PPOConfig(hidden=(32, 16)), dtype=D64)
    with pytest.raises(P.DigestMismatch):
        b.load(ref)


def test_nonfinite_loss_rolls_back(z):
    a = _agent(z)
    before = [p.detach().clone() for p in a.net.params()]
    obs, act, lp, v, adv, ret = _batch(z)
    ret = ret.clone()
    ret[0] = float("nan")
    with pytest.raises(P.NonFiniteLoss):
        a.update(obs, act, lp, v, adv, ret)
    for p, b in zip(a.net.params(), before):
        assert torch.equal(p.detach(), b)


class BanditEnv:
    """Reference tests/test_ppo.py:223-243: reward = -sum (a - 0.3)^2."""
    obs_dim, act_dim = 1, 2

    class _Cfg:
        num_envs = 64

    def __init__(self):
        self.config = self._Cfg()

    def reset(self, env_indices=None):
        return torch.zeros((64, 1), dtype=D64)

    def step(self, actions):
        from paper_2108_10470_b200.envs import StepOutput
        a = torch.clamp(actions, -1, 1)
        return StepOutput(torch.zeros((64, 1), dtype=D64), -((a - 0.3) ** 2).sum(-1),
                          torch.zeros(64, dtype=torch.bool), {})


def test_policy_improves_on_bandit(tmp_path):
    env = BanditEnv()
    cfg = P.PPOConfig(hidden=(16,), lr=5e-3, minibatch_size=256, gamma=0.0, lam=0.0)
    agent = P.PPO(1, 2, cfg, seed=0, dtype=D64)
    hist = P.train(env, agent, iterations=60, horizon=8, metrics_path=str(tmp_path / "m.csv"),
                   checkpoint_path=str(tmp_path / "c.bin"))
    early = np.mean([h["mean_reward"] for h in hist[:5]])
    late = np.mean([h["mean_reward"] for h in hist[-5:]])
    assert late > early + 0.3
    mu = agent.net.actor(torch.zeros((1, 1), dtype=D64))
    assert float((mu - 0.3).abs().max()) < 0.2
    lines = (tmp_path / "m.csv").read_text().splitlines()
    assert lines[0] == "iteration,env_steps,mean_reward,loss,pg_loss,v_loss,kl,lr,wall_clock_s"
    assert len(lines) == 61 and lines[-1].startswith("60,30720,")
    assert (tmp_path / "c.bin").exists()


# ------------------------------------------------------ data parallel (gloo)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dp_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(os.path.join(GOLD, "ppo.npz"))
    a = _agent(z)
    batch = _batch(z)
    N = batch[0].shape[0]
    lo, hi = rank * N // world, (rank + 1) * N // world
    a.config.minibatch_size = hi - lo          # one minibatch per rank = the global batch
    st = a.update(*(x[lo:hi] for x in batch))
    if rank == 0:
        np.savez(out_path, lr=st["lr"], **{f"p{i}": p.detach().numpy() for i, p in enumerate(a.net.params())})
    dist.destroy_process_group()


def test_data_parallel_update_equals_single_process(tmp_path):
    """Gradient all-reduce + global advantage normalisation + global KL: two
    ranks on the two halves of the batch produce the parameters of the
    reference's single-process full-batch update."""
    out = str(tmp_path / "dp.npz")
    mp.spawn(_dp_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    z = np.load(os.path.join(GOLD, "ppo.npz"))
    n = len([k for k in z.files if k.startswith("param1_")])
    for i in range(n):
        np.testing.assert_allclose(got[f"p{i}"], z[f"param1_{i}"], rtol=1e-9, atol=1e-12)
    assert float(got["lr"]) == pytest.approx(float(z["update_lr"][0]))
