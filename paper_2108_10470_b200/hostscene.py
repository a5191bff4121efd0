"""`HostScene`: the reference's NumPy `Scene` protocol over the B200 step.

The reference's task layer (`EnvBatch`, `SimBuffers`, `DomainRandomizer`,
/root/reference/pkg/src/batchsim/envs.py:72-200, buffers.py:47-225,
randomize.py:86-189) is NumPy code that reads and writes the scene's arrays
in place: ``scene.root_state.copy()`` (envs.py:137), ``s.pos[base] = rows``
in WORLD frame (buffers.py:145), ``scene.nonfinite[envs]`` (envs.py:149),
``scene.mu_static[envs] = ...`` (randomize.py).  The device `Scene`
(scene.py) keeps its state as CUDA tensors with env-local positions, so that
code cannot drive it directly.  `HostScene` is the adapter a maintainer puts
behind the one-line swap at envs.py:86-91:

* every array attribute of the reference `Scene` (physics.py:147-355) is a
  float64 (or the reference's integer / bool) NumPy array of the reference
  shape, positions and friction anchors in WORLD frame;
* `step()` pushes the host arrays the step reads (body poses / velocities,
  anchors, DOF state, controls, DOF modes, per-env parameters, the poison
  flags) to the device, runs one `bsim_step` launch, and pulls back what a
  step writes (physics.py:538-596 + refresh_buffers 1037-1071);
* `forward_kinematics(env_mask, actors)` (physics.py:366-425) does the same
  around `bsim_forward_kinematics`.

The conversion world <-> env-local happens in float64 on the host, so with
``precision="fp64"`` the reference's own env code over `HostScene` matches
the reference `Scene` at the fp64 parity bound (tests/test_gpu_dropin.py).
This is the compatibility path for unmodified NumPy task code; the fused
device task layer (`envs.make_env`) is the fast path.
"""

from __future__ import annotations

import numpy as np
import torch

from .scene import ContactPoint, Scene

__all__ = ["HostScene", "ContactPoint"]

# per-env parameter arrays the reference's DomainRandomizer may rewrite
_PARAMS = ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static", "mu_dynamic",
           "joint_stiffness", "joint_damping", "joint_armature", "joint_friction", "joint_limit_lo",
           "joint_limit_hi", "plane_off", "plane_rad", "pair_off", "pair_rad")
_CONTROLS = ("ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
             "ctrl_body_torque")
_OUTPUTS = ("root_state", "body_state", "dof_state", "net_contact", "dof_force", "sensor_forces")


class HostScene:
    """Reference `Scene` (physics.py:140) with NumPy arrays, stepped on a B200."""

    def __init__(self, models, num_envs, params=None, spacing=4.0, ground=True, env_origins=None,
                 precision="fp64", device=None):
        self.dev = d = Scene(models, num_envs, params, spacing, ground, env_origins, device=device,
                             precision=precision)
        self.models, self.num_envs, self.params, self.ground = d.models, d.num_envs, d.params, d.ground
        for k in ("actors_per_env", "bodies_per_env", "dofs_per_env", "sensors_per_env", "num_bodies",
                  "num_dofs", "num_actors", "actor_body_offset", "actor_dof_offset", "env_body_base",
                  "env_dof_base", "sensor_body"):
            setattr(self, k, getattr(d, k))
        self.env_origins = d.env_origins_host.copy()
        self.body_env = np.repeat(np.arange(self.num_envs), self.bodies_per_env)
        self.step_count = 0
        self.dof_mode = d.dof_mode.cpu().numpy().astype(np.int8)
        for k in _PARAMS + _CONTROLS:
            setattr(self, k, self._host(getattr(d, k)))
        self._pull_state()

    # ------------------------------------------------------------ transfer
    @staticmethod
    def _host(t):
        return t.detach().double().cpu().numpy().copy()

    def _put(self, t, a):
        t.copy_(torch.from_numpy(np.ascontiguousarray(a)).to(t.device, t.dtype))

    def _pull_state(self):
        d = self.dev
        q = self._host(d.body_q)
        self.pos = q[:, 0:3] + self.env_origins[self.body_env]
        self.quat, self.linvel, self.angvel = q[:, 3:7].copy(), q[:, 7:10].copy(), q[:, 10:13].copy()
        self._friction_anchor = self._host(d._friction_anchor) + self.env_origins[None]
        for k in _OUTPUTS:
            setattr(self, k, self._host(getattr(d, k)))
        self.nonfinite = d.nonfinite.cpu().numpy().astype(bool)

    def _push_state(self):
        d = self.dev
        q = np.concatenate([self.pos - self.env_origins[self.body_env], self.quat, self.linvel, self.angvel], 1)
        self._put(d.body_q, q)
        self._put(d._friction_anchor, self._friction_anchor - self.env_origins[None])
        self._put(d.dof_state, self.dof_state)
        self._put(d.nonfinite, self.nonfinite)
        self._put(d.dof_mode, self.dof_mode)
        for k in _PARAMS + _CONTROLS:
            self._put(getattr(d, k), getattr(self, k))

    # ------------------------------------------------------------ protocol
    def step(self):
        """physics.py:538-596 on the device; host arrays are current on return."""
        self._push_state()
        self.dev.step()
        self.dev.fetch_results()
        self._pull_state()
        self.step_count += 1

    def forward_kinematics(self, env_mask=None, actors=None):
        """physics.py:366-425 for the selected envs / actors (world-frame roots in, links out)."""
        self._push_state()
        self.dev.forward_kinematics(env_mask=env_mask, actors=actors)
        self.dev.fetch_results()
        self._pull_state()

    def refresh_buffers(self):
        self._push_state()
        self.dev.refresh_buffers()
        self.dev.fetch_results()
        self._pull_state()

    def read_dof_states(self):
        self.refresh_buffers()

    def collide(self):
        self._push_state()
        return self.dev.collide()

    def clear_nonfinite(self, env_indices):          # physics.py:1089-1090
        self.nonfinite[env_indices] = False

    def close(self):
        self.dev.close()

