"""Golden vectors for the PPO caller, produced by the REFERENCE
(/root/reference/pkg/src/batchsim/ppo.py; run here, the reference does not
travel to the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ppo_golden.py

Writes tests/golden/ppo.npz (+ ppo_ckpt.bin, a reference-written checkpoint):
  * GAE on a random (T, E) rollout with episode cuts   (ppo.py:215-229)
  * loss stats and gradients of ActorCritic(seed 0)      (ppo.py:159-209)
  * one reference PPO.update (1 epoch, full batch) and its parameters after
  * Adam moments after two steps                         (ppo.py:234-251)
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from batchsim.ppo import PPO, Adam, PPOConfig, gae_advantages  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(7)
    arrays = {}
    # ---- GAE
    T, E = 12, 9
    rew = rng.normal(size=(T, E))
    val = rng.normal(size=(T, E))
    dones = (rng.uniform(size=(T, E)) < 0.15).astype(np.float64)
    last = rng.normal(size=E)
    adv, ret = gae_advantages(rew, val, dones, last, 0.99, 0.95)
    arrays.update(gae_rewards=rew, gae_values=val, gae_dones=dones, gae_last=last, gae_adv=adv, gae_ret=ret)

    # ---- loss + grads (small net so the fixture stays small)
    cfg = PPOConfig(hidden=(32, 16), minibatch_size=64, epochs=1, entropy_coef=0.01)
    obs_dim, act_dim, N = 7, 3, 64
    agent = PPO(obs_dim, act_dim, cfg, seed=3)
    agent.net.log_std[:] = rng.normal(scale=0.3, size=act_dim)
    obs = rng.normal(size=(N, obs_dim))
    act = rng.normal(size=(N, act_dim))
    mu, _ = agent.net.actor.forward(obs)
    logp_old = agent.net.log_prob(mu, act) + rng.normal(scale=0.2, size=N)
    v_old = agent.net.value(obs) + rng.normal(scale=0.3, size=N)
    advs = rng.normal(size=N)
    rets = rng.normal(size=N)
    stats, grads = agent.net.loss_and_grads(obs, act, logp_old, v_old, advs, rets)
    params0 = [p.copy() for p in agent.net.params()]
    for i, p in enumerate(params0):
        arrays[f"param0_{i}"] = p
    for i, g in enumerate(grads):
        arrays[f"grad_{i}"] = g
    arrays.update(obs=obs, act=act, logp_old=logp_old, v_old=v_old, adv=advs, ret=rets,
                  stats=np.array([stats[k] for k in ("loss", "pg_loss", "v_loss", "entropy", "kl")]))
    agent.save(os.path.join(OUT, "ppo_ckpt.bin"))

    # ---- one full-batch update (1 epoch, minibatch = N: order-independent)
    st = agent.update(obs, act, logp_old, v_old, advs, rets)
    for i, p in enumerate(agent.net.params()):
        arrays[f"param1_{i}"] = p.copy()
    arrays["update_lr"] = np.array([st["lr"]])

    # ---- Adam
    ps = [rng.normal(size=(4, 3)), rng.normal(size=5)]
    opt = Adam(ps, lr=1e-2)
    g1 = [rng.normal(size=(4, 3)), rng.normal(size=5)]
    g2 = [rng.normal(size=(4, 3)), rng.normal(size=5)]
    arrays.update(adam_p0a=ps[0].copy(), adam_p0b=ps[1].copy(), adam_g1a=g1[0], adam_g1b=g1[1],
                  adam_g2a=g2[0], adam_g2b=g2[1])
    opt.step(ps, g1)
    opt.step(ps, g2)
    arrays.update(adam_p2a=ps[0], adam_p2b=ps[1])
    np.savez_compressed(os.path.join(OUT, "ppo.npz"), **arrays)
    print("wrote ppo.npz, ppo_ckpt.bin")


if __name__ == "__main__":
    main()
