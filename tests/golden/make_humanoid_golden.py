"""Golden vectors for the authored humanoid (BASELINE.json config
"Humanoid"), produced by the REFERENCE (run here; the reference does not
travel to the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_humanoid_golden.py

The reference bundles no humanoid, so the model is the
authored JSON document `paper_2108_10470_b200.models.humanoid_doc()` (plain
data in the reference schema) loaded by the reference's own `load_model`:
  * humanoid_walk / humanoid_drop: reference `Scene.step()` traces
    (physics.py:538-592) with capsule + sphere plane slots and 21 PD hinges;
  * env_humanoid: the reference `QuadrupedEnv` task (envs.py:359-478: obs
    layout, locomotion_reward, reset law) run on the humanoid with its own
    rest height and termination height -- the same task the GPU
    `HumanoidEnv` implements.
"""

from __future__ import annotations

import os
import sys
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
for p in (REF, HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

from batchsim.envs import EnvBatch, EnvConfig, QuadrupedEnv  # noqa: E402
from batchsim.model import load_model  # noqa: E402
from batchsim.physics import SimParams  # noqa: E402

import make_golden as G  # noqa: E402
from paper_2108_10470_b200.models import HUMANOID_REST_HEIGHT, humanoid_doc  # noqa: E402

TERMINATION_HEIGHT = 0.8


class HumanoidRefEnv(QuadrupedEnv):
    """Reference QuadrupedEnv algorithm with the humanoid's constants."""

    name = "humanoid"
    obs_dim = 87
    act_dim = 21

    def __init__(self, config):
        EnvBatch.__init__(self, replace(config, sim_dt=1.0 / 120.0, control_dt=1.0 / 60.0))

    def _model(self):
        return load_model(humanoid_doc())

    def _post_reset(self, envs):
        super()._post_reset(envs)
        self.reward_params.termination_height = TERMINATION_HEIGHT

    def _reset_envs(self, envs, rngs):
        # envs.py:404-419 with the humanoid's rest height
        E = self.config.num_envs
        root = self.scene.root_state.copy()
        root[:, 0:3] -= self.scene.env_origins
        dof = self.scene.dof_state.copy()
        dview = dof.reshape(E, self.act_dim, 2)
        for e, rng in zip(envs, rngs):
            root[e] = 0.0
            root[e, 2] = HUMANOID_REST_HEIGHT + 0.02
            yaw = rng.uniform(-0.1, 0.1)
            root[e, 3:7] = [0.0, 0.0, np.sin(yaw / 2), np.cos(yaw / 2)]
            dview[e, :, 0] = rng.uniform(-0.1, 0.1, self.act_dim)
            dview[e, :, 1] = 0.0
        root[:, 0:3] += self.scene.env_origins
        self.buffers.set_root_state(root, envs)
        self.buffers.set_dof_state(dof, envs)


def env_case(E=6, steps=28):
    env = HumanoidRefEnv(EnvConfig(num_envs=E, seed=3, episode_length=25))
    rng = np.random.default_rng(99)
    rec = {k: [] for k in ("actions", "obs", "reward", "done", "timeout", "root_state", "dof_state", "pos",
                           "quat", "linvel", "angvel", "_friction_anchor", "sensor_forces", "dof_force",
                           "ctrl_dof_pos_target", "episode_steps", "reset_count", "extra_before",
                           "extra_after")}
    obs0 = env.reset()
    for t in range(steps):
        a = rng.uniform(-1.2, 1.2, (E, env.act_dim))
        if t == 5:      # knock env 2 down so the termination path fires
            root = env.scene.root_state.copy()
            root[2, 2] = 0.5
            env.buffers.set_root_state(root, [2])
        rec["extra_before"].append(np.array(env.potentials, copy=True))
        pre = G.snapshot(env.scene, ("pos", "quat", "linvel", "angvel", "_friction_anchor", "root_state",
                                     "dof_state", "sensor_forces", "dof_force"))
        for k, v in pre.items():
            rec[k].append(v)
        rec["episode_steps"].append(env.episode_steps.copy())
        rec["reset_count"].append(env.reset_count.copy())
        out = env.step(a)
        rec["actions"].append(a)
        rec["obs"].append(out.obs.copy())
        rec["reward"].append(out.reward.copy())
        rec["done"].append(out.done.copy())
        rec["timeout"].append(out.info["timeout"].copy())
        rec["ctrl_dof_pos_target"].append(env.scene.ctrl_dof_pos_target.copy())
        rec["extra_after"].append(np.array(env.potentials, copy=True))
    arrays = {k: np.stack(v) for k, v in rec.items()}
    arrays["obs0"] = obs0
    arrays["env_origins"] = env.scene.env_origins.copy()
    meta = {"kind": "env", "task": "humanoid", "num_envs": E, "steps": steps, "seed": 3, "episode_length": 25}
    G.save("env_humanoid", meta, arrays)


def main():
    dt = 1.0 / 120.0
    doc = humanoid_doc()
    # stand, settle for 30 steps, then random PD targets
    G.physics_case("humanoid_walk", [doc], 6, SimParams(dt=dt), 8,
                   G.reset_walkers(HUMANOID_REST_HEIGHT + 0.02, vscale=0.3), G.rng_targets(0.5, 21), warmup=30)
    # a fall: tilted drop with large joint offsets (many capsule / sphere slots touch down)
    G.physics_case("humanoid_drop", [doc], 6, SimParams(dt=dt), 10,
                   G.reset_walkers(HUMANOID_REST_HEIGHT + 0.3, yaw=1.0, qscale=0.6, vscale=1.5, seed=8),
                   G.rng_targets(0.6, 22), warmup=45)
    env_case()
    print("wrote humanoid_walk, humanoid_drop, env_humanoid")


if __name__ == "__main__":
    main()
