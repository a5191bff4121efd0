"""Golden traces at BASELINE.json scale, produced by the REFERENCE (run here;
the reference does not travel to the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scale_golden.py [task ...]

For the Ant analog (`quadruped`, BASELINE config 1) and the ANYmal analog
(`quadruped-anymal-obs`, config 3) at 4096 envs, the reference `EnvBatch`
(envs.py:178-200) runs 20 control steps FREE from construction (seed 0,
episode_length 12 so every env times out and auto-resets at step 12, and
every 4th env knocked down to z = 0.1 through `set_root_state` before step 5
so a quarter of the batch terminates there), actions U(-1, 1) from `np.random.default_rng(0)` per
step as in the reference bench (cli.py:129-140).  After every step the
post-step state and the env outputs are recorded for a fixed 1/32 sample of
the envs (every 32nd env: 128 rows) -- the whole batch would be ~90 MB.

Tests pin the oracle to these traces at 1e-7 (the oracle then stands in for
the reference on all 4096 envs) and compare the CUDA path against both.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
if REF not in sys.path:
    sys.path.insert(0, REF)

from batchsim.envs import make_env  # noqa: E402

E, STEPS, STRIDE, EPISODE = 4096, 20, 32, 12
KNOCK_STEP, KNOCK = 5, np.arange(1, 4096, 4)
CASES = (("quadruped", "scale_ant_4096", "potentials"),
         ("quadruped-anymal-obs", "scale_anymal_4096", "commands"),
         # BASELINE config 2's model: the reference QuadrupedEnv algorithm on the
         # authored humanoid (make_humanoid_golden.HumanoidRefEnv), knocked to z 0.5
         ("humanoid", "scale_humanoid_4096", "potentials"))
KNOCK_Z = {"quadruped": 0.1, "quadruped-anymal-obs": 0.1, "humanoid": 0.5}


def _make(task):
    if task == "humanoid":
        sys.path.insert(0, HERE)
        from batchsim.envs import EnvConfig
        from make_humanoid_golden import HumanoidRefEnv
        return HumanoidRefEnv(EnvConfig(num_envs=E, seed=0, episode_length=EPISODE))
    return make_env(task, num_envs=E, seed=0, episode_length=EPISODE)


def sample_rows(idx, per_env):
    return (idx[:, None] * per_env + np.arange(per_env)).ravel()


def main(only=None):
    for task, name, extra in CASES:
        if only and task not in only:
            continue
        t0 = time.time()
        env = _make(task)
        s = env.scene
        B, D, S = s.bodies_per_env, s.dofs_per_env, s.sensors_per_env
        idx = np.arange(0, E, STRIDE)
        rb, rd, rs = sample_rows(idx, B), sample_rows(idx, D), sample_rows(idx, S)
        rng = np.random.default_rng(0)
        rec = {k: [] for k in ("obs", "reward", "done", "timeout", "body_state", "dof_state", "net_contact",
                               "sensor_forces", "dof_force", "friction_anchor", "episode_steps",
                               "reset_count", "extra", "ctrl_dof_pos_target")}
        arrays = {"sample": idx, "env_origins": s.env_origins[idx].copy(),
                  "obs0": env._observe()[idx].copy(), "extra0": np.array(getattr(env, extra))[idx].copy(),
                  "body_state0": s.body_state[rb].copy(), "dof_state0": s.dof_state[rd].copy()}
        for t in range(STEPS):
            a = rng.uniform(-1.0, 1.0, (E, env.act_dim))
            if t == KNOCK_STEP:
                # knock every 4th env down (world z 0.1, below both tasks' termination
                # heights) through the buffer API, as the reference's own env trace does
                root = s.root_state.copy()
                root[KNOCK, 2] = KNOCK_Z[task]
                env.buffers.set_root_state(root, KNOCK)
            out = env.step(a)
            rec["obs"].append(out.obs[idx])
            rec["reward"].append(out.reward[idx])
            rec["done"].append(out.done[idx])
            rec["timeout"].append(out.info["timeout"][idx])
            rec["body_state"].append(s.body_state[rb].copy())
            rec["dof_state"].append(s.dof_state[rd].copy())
            rec["net_contact"].append(s.net_contact[rb].copy())
            rec["sensor_forces"].append(s.sensor_forces[rs].copy())
            rec["dof_force"].append(s.dof_force[rd].copy())
            rec["friction_anchor"].append(s._friction_anchor[:, idx].copy())
            rec["episode_steps"].append(env.episode_steps[idx].copy())
            rec["reset_count"].append(env.reset_count[idx].copy())
            rec["extra"].append(np.array(getattr(env, extra))[idx].copy())
            rec["ctrl_dof_pos_target"].append(s.ctrl_dof_pos_target[rd].copy())
            # full-batch masks are small: keep them whole (bit-exactness at scale)
            arrays.setdefault("done_all", []).append(out.done.copy())
            arrays.setdefault("timeout_all", []).append(out.info["timeout"].copy())
            print(f"{name}: step {t} done={int(out.done.sum())} ({time.time() - t0:.0f}s)", flush=True)
        arrays.update({k: np.stack(v) for k, v in rec.items()})
        arrays["done_all"] = np.stack(arrays["done_all"])
        arrays["timeout_all"] = np.stack(arrays["timeout_all"])
        meta = {"kind": "scale_env", "task": task, "num_envs": E, "steps": STEPS, "seed": 0, "stride": STRIDE,
                "episode_length": EPISODE, "actions": "np.random.default_rng(0).uniform(-1, 1, (E, A)) per step",
                "extra": extra, "knock_step": KNOCK_STEP,
                "knock": f"np.arange(1, 4096, 4), world z = {KNOCK_Z[task]}"}
        import json
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(meta), **arrays)
        print(f"wrote {name}.npz in {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or None)     # optionally only the named tasks
