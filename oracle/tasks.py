"""CPU ORACLE task layer -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference env layer for the benchmarked
locomotion tasks, driven over `OracleScene` (the C restatement of
`Scene.step`):

* `EnvBatch.step` / `reset` / `_observe`  /root/reference/pkg/src/batchsim/envs.py:117-200
* `QuadrupedEnv` (Ant analog)              envs.py:359-478
* `AnymalObsEnv` (ANYmal analog, flat)     envs.py:484-565
* humanoid: the QuadrupedEnv algorithm with the humanoid's rest and
  termination heights (tests/golden/make_humanoid_golden.py:41-78)
* `locomotion_reward` / `anymal_reward`    rewards.py:78-112 / 129-158
* indexed `set_root_state` / `set_dof_state` (write rows -> FK over the
  touched envs -> repack)                  buffers.py:109-178

Resets draw from `np.random.default_rng([seed, env, reset_count])`
(envs.py:129-133); `env` is the GLOBAL env id (`env_offset + e`), which for
an unsharded batch is the reference's own index.  Pinned against the
reference's env traces (tests/test_oracle_golden.py::test_oracle_env_*).

Only tests/, `__graft_entry__.smoke()` and bench.py's CPU legs use this.
"""

from __future__ import annotations

import numpy as np

from .oracle import OracleScene

TASK_SPECS = {
    # name: (model builder, act_dim, obs_dim, action_scale, rest height, termination height)
    "quadruped": ("quadruped", 8, 60, 0.6, 0.35, 0.26),
    "quadruped-anymal-obs": ("quadruped12", 12, 48, 0.5, 0.32, None),
    "humanoid": ("humanoid", 21, 87, 0.6, 1.42, 0.8),
}


def _cross(a, b):
    return np.cross(a, b)


def quat_rotate(q, v):                       # spatial.py:57-64
    u, w = q[..., :3], q[..., 3:4]
    t = 2.0 * _cross(u, v)
    return v + w * t + _cross(u, t)


def quat_rotate_inverse(q, v):               # spatial.py:67-68
    qc = np.concatenate([-q[..., :3], q[..., 3:4]], axis=-1)
    return quat_rotate(qc, v)


def dof_limits(model):                       # envs.py:27-35
    lo, hi = [], []
    for j in model.joints:
        for _ in range(j.dof_count):
            lo.append(j.limits[0] if j.limits else -np.inf)
            hi.append(j.limits[1] if j.limits else np.inf)
    return np.asarray(lo, float), np.asarray(hi, float)


def locomotion_reward(torso, target, up_proj, heading_proj, actions, qpos, qvel, lo, hi, strength,
                      prev_potential, dt, termination_height):
    """rewards.py:78-112 with LocomotionRewardParams defaults (rewards.py:16-27)."""
    dist = np.linalg.norm(target - torso, axis=-1)
    potential = -dist / dt
    r = potential - prev_potential
    h = torso[:, 2]
    r = r + np.where(h >= termination_height, 0.5, 0.0)
    r = r + np.where(h <= termination_height, -1.0, 0.0)
    r = r + np.where(up_proj > 0.93, 0.1, 0.0)
    r = r + 0.5 * np.where(heading_proj >= 0.8, 1.0, heading_proj / 0.8)
    r = r - 0.005 * np.sum(actions ** 2, axis=-1)
    r = r + 0.05 * np.sum(actions * strength * qvel, axis=-1)
    limited = np.isfinite(lo) & np.isfinite(hi)
    span = np.where(limited, hi - lo, 1.0)
    frac = (qpos - lo) / span
    near = ((frac < 0.01) | (frac > 0.99)) & limited
    r = r - 0.1 * np.sum(near, axis=-1)
    return r, potential


def anymal_reward_flat(lin_b, ang_b, cmd, torques, dt):
    """rewards.py:129-148 (variant "flat", AnymalRewardParams defaults)."""
    err_xy = np.sum((cmd[:, 0:2] - lin_b[:, 0:2]) ** 2, axis=-1)
    err_yaw = (cmd[:, 2] - ang_b[:, 2]) ** 2
    phi = lambda x: np.exp(-x / 0.25)  # noqa: E731  rewards.py:120-126
    return 1.0 * dt * phi(err_xy) + 0.5 * dt * phi(err_yaw) - 0.00002 * dt * np.sum(torques ** 2, axis=-1)


class OracleEnv:
    """Reference `EnvBatch` semantics for one locomotion task over the C oracle."""

    def __init__(self, task, num_envs, seed=0, episode_length=1000, env_offset=0, total_envs=None,
                 threads=1, scene=None):
        from paper_2108_10470_b200 import models as M
        from paper_2108_10470_b200.layout import SceneLayout
        from paper_2108_10470_b200.params import SimParams
        if task not in TASK_SPECS:
            raise KeyError(task)
        self.task = task
        model_name, self.act_dim, self.obs_dim, self.action_scale, self.rest_height, term = TASK_SPECS[task]
        self.termination_height = term
        self.model = getattr(M, model_name)()
        self.num_envs = E = int(num_envs)
        self.seed, self.episode_length = int(seed), int(episode_length)
        self.env_offset = int(env_offset)
        total = E + self.env_offset if total_envs is None else int(total_envs)
        self.control_dt, self.decimation = 1.0 / 60.0, 2
        if scene is None:
            origins = SceneLayout([self.model]).default_env_origins(total)[self.env_offset:self.env_offset + E]
            scene = OracleScene([self.model], E, SimParams(dt=1.0 / 120.0), env_origins=origins, threads=threads)
        self.scene = scene
        self.episode_steps = np.zeros(E, np.int64)
        self.reset_count = np.zeros(E, np.int64)
        self.actions = np.zeros((E, self.act_dim))
        self.dof_lower, self.dof_upper = dof_limits(self.model)
        self.motor_strength = np.ones((E, self.act_dim))
        self.potentials = np.zeros(E)
        self.commands = np.zeros((E, 3))
        self.reset()

    # ------------------------------------------------------------ buffers.py restated
    def _repack(self, envs):                                  # buffers.py:109-123
        s = self.scene
        B = s.bodies_per_env
        rows = (envs[:, None] * B + np.arange(B)).ravel()
        s.body_state[rows] = np.concatenate([s.pos[rows], s.quat[rows], s.linvel[rows], s.angvel[rows]], 1)
        s.root_state[envs] = s.body_state[envs * B]

    def _fk(self, envs):
        mask = np.zeros(self.num_envs, bool)
        mask[envs] = True
        self.scene.forward_kinematics(env_mask=mask, actors={0})
        self._repack(envs)

    def set_root_state(self, rows_local, envs):               # buffers.py:127-151
        """rows_local (len(envs), 13): env-local root rows of actor 0."""
        s = self.scene
        q = rows_local[:, 3:7]
        rows = rows_local.copy()
        rows[:, 3:7] = q / np.linalg.norm(q, axis=-1, keepdims=True)
        rows[:, 0:3] += s.env_origins[envs]
        s.root_state[envs] = rows
        base = envs * s.bodies_per_env
        s.pos[base], s.quat[base], s.linvel[base], s.angvel[base] = (rows[:, 0:3], rows[:, 3:7], rows[:, 7:10],
                                                                     rows[:, 10:13])
        self._fk(envs)

    def set_dof_state(self, dof_rows, envs):                  # buffers.py:154-178
        """dof_rows (len(envs), D, 2)."""
        s = self.scene
        D = s.dofs_per_env
        rows = (envs[:, None] * D + np.arange(D)).ravel()
        s.dof_state[rows] = dof_rows.reshape(-1, 2)
        self._fk(envs)

    # ------------------------------------------------------------ EnvBatch
    def local_root(self):                                     # envs.py:135-139
        root = self.scene.root_state.copy()
        root[:, 0:3] -= self.scene.env_origins
        return root

    def dof_view(self):
        return self.scene.dof_state.reshape(self.num_envs, -1, 2)

    def _env_rng(self, e):                                    # envs.py:129-133 (global env id)
        return np.random.default_rng([self.seed, int(self.env_offset + e), int(self.reset_count[e])])

    def _reset_envs(self, envs, rngs):                        # envs.py:404-419 / 536-549
        n = len(envs)
        root = np.zeros((n, 13))
        root[:, 2] = self.rest_height + 0.02
        dof = np.zeros((n, self.act_dim, 2))
        for i, rng in enumerate(rngs):
            if self.task == "quadruped-anymal-obs":
                root[i, 6] = 1.0
            else:
                yaw = rng.uniform(-0.1, 0.1)
                root[i, 3:7] = [0.0, 0.0, np.sin(yaw / 2), np.cos(yaw / 2)]
            dof[i, :, 0] = rng.uniform(-0.1, 0.1, self.act_dim)
        self.set_root_state(root, envs)
        self.set_dof_state(dof, envs)

    def _post_reset(self, envs):                              # envs.py:383-391 / 529-534
        if self.task == "quadruped-anymal-obs":
            for e in envs:
                rng = np.random.default_rng([self.seed, int(self.env_offset + e), int(self.reset_count[e]), 0xC])
                self.commands[e] = rng.uniform([-1.0, -1.0, -1.0], [1.0, 1.0, 1.0])
            return
        root = self.local_root()
        dist = np.linalg.norm(self._targets()[envs] - root[envs, 0:3], axis=-1)
        self.potentials[envs] = -dist / self.control_dt

    def _targets(self):
        t = np.zeros((self.num_envs, 3))
        t[:, 0] = 1000.0                                      # QuadrupedEnv.target_x
        return t

    def reset(self, env_indices=None):                        # envs.py:141-166
        E = self.num_envs
        envs = np.arange(E) if env_indices is None else np.atleast_1d(np.asarray(env_indices, np.int64))
        if envs.size == 0:
            return self._compute_obs()
        poisoned = envs[self.scene.nonfinite[envs]]
        if poisoned.size:
            self.scene.clear_nonfinite(poisoned)
        rngs = [self._env_rng(e) for e in envs]
        self._reset_envs(envs, rngs)
        self.episode_steps[envs] = 0
        self.reset_count[envs] += 1
        self.actions[envs] = 0.0
        self._post_reset(envs)
        return self._compute_obs()

    def _frame(self):                                         # envs.py:429-443
        root = self.local_root()
        quat = root[:, 3:7]
        E = len(root)
        lin_b = quat_rotate_inverse(quat, root[:, 7:10])
        ang_b = quat_rotate_inverse(quat, root[:, 10:13])
        up = quat_rotate(quat, np.broadcast_to([0.0, 0.0, 1.0], (E, 3)))
        heading = quat_rotate(quat, np.broadcast_to([1.0, 0.0, 0.0], (E, 3)))
        to_dir = (self._targets() - root[:, 0:3])[:, 0:2]
        to_dir = to_dir / np.maximum(np.linalg.norm(to_dir, axis=-1, keepdims=True), 1e-9)
        heading_proj = np.sum(heading[:, 0:2] * to_dir, axis=-1)
        return root, lin_b, ang_b, up[:, 2], heading_proj

    def _compute_obs(self):
        E = self.num_envs
        d = self.dof_view()
        if self.task == "quadruped-anymal-obs":                # envs.py:551-564
            root = self.local_root()
            quat = root[:, 3:7]
            lin_b = quat_rotate_inverse(quat, root[:, 7:10])
            ang_b = quat_rotate_inverse(quat, root[:, 10:13])
            grav = quat_rotate_inverse(quat, np.broadcast_to([0.0, 0.0, -1.0], (E, 3)))
            return np.concatenate([lin_b, ang_b, grav, self.commands, d[:, :, 0], d[:, :, 1] * 0.05,
                                   self.actions], axis=-1)
        root, lin_b, ang_b, up_z, heading_proj = self._frame()  # envs.py:445-465
        x, y, z, w = root[:, 3], root[:, 4], root[:, 5], root[:, 6]
        yaw = np.arctan2(2 * (w * z + x * y), 1 - 2 * (y * y + z * z))
        roll = np.arctan2(2 * (w * x + y * z), 1 - 2 * (x * x + y * y))
        to_target = self._targets() - root[:, 0:3]
        angle_to = np.arctan2(to_target[:, 1], to_target[:, 0]) - yaw
        angle_to = np.arctan2(np.sin(angle_to), np.cos(angle_to))
        span = self.dof_upper - self.dof_lower
        dof_scaled = 2.0 * (d[:, :, 0] - self.dof_lower) / span - 1.0
        sensors = self.scene.sensor_forces.reshape(E, -1) * 0.01
        return np.concatenate([root[:, 2:3], lin_b, ang_b, yaw[:, None], roll[:, None], angle_to[:, None],
                               up_z[:, None], heading_proj[:, None], dof_scaled, d[:, :, 1] * 0.05, sensors,
                               self.actions], axis=-1)

    def _compute_reward_done(self):
        E = self.num_envs
        if self.task == "quadruped-anymal-obs":                # envs.py:566-580
            root = self.local_root()
            quat = root[:, 3:7]
            lin_b = quat_rotate_inverse(quat, root[:, 7:10])
            ang_b = quat_rotate_inverse(quat, root[:, 10:13])
            torques = self.scene.dof_force.reshape(E, self.act_dim)
            reward = anymal_reward_flat(lin_b, ang_b, self.commands, torques, self.control_dt)
            up_z = quat_rotate(quat, np.broadcast_to([0.0, 0.0, 1.0], (E, 3)))[:, 2]
            return reward, (up_z < 0.3) | (root[:, 2] < 0.18)
        root, _, _, up_z, heading_proj = self._frame()         # envs.py:467-476
        d = self.dof_view()
        reward, self.potentials = locomotion_reward(
            root[:, 0:3], self._targets(), up_z, heading_proj, self.actions, d[:, :, 0], d[:, :, 1],
            self.dof_lower, self.dof_upper, self.motor_strength, self.potentials, self.control_dt,
            self.termination_height)
        return reward, root[:, 2] <= self.termination_height

    def apply_actions(self, actions):                         # envs.py:421-424 / 547-550
        self.scene.ctrl_dof_pos_target[:] = (self.action_scale * actions).reshape(-1)

    def step(self, actions):                                  # envs.py:178-200
        actions = np.clip(np.asarray(actions, np.float64), -1.0, 1.0)
        if actions.shape != (self.num_envs, self.act_dim):
            raise ValueError(f"actions must have shape ({self.num_envs}, {self.act_dim})")
        self.actions = actions
        self.apply_actions(actions)
        for _ in range(self.decimation):
            self.scene.step()
        self.episode_steps += 1
        reward, done = self._compute_reward_done()
        timeout = self.episode_steps >= self.episode_length
        poisoned = self.scene.nonfinite.copy()
        done = done | timeout | poisoned
        reward = np.where(poisoned, 0.0, reward)
        obs = self._compute_obs()
        if np.any(done):
            idx = np.nonzero(done)[0]
            fresh = self.reset(idx)
            obs[idx] = fresh[idx]
        return obs, reward, done.copy(), {"timeout": timeout, "poisoned": poisoned}
