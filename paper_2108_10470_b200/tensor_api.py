"""Gym-style tensor API over a GPU Scene (the interface named by the north
star; Isaac Gym's `gym.acquire_*_tensor` / `set_*_tensor` / `simulate` /
`fetch_results` family).

Every `acquire_*` returns the scene's canonical device tensor (zero-copy,
the same object on every call, as buffers.py:55-78); setters copy into the
canonical storage (indexed setters go through SimBuffers with the
reference's validation and error classes); `simulate` launches the fused
step asynchronously and `fetch_results` waits for it.
"""

from __future__ import annotations

import torch

from .buffers import SimBuffers


class TensorAPI:
    def __init__(self, scene):
        self.scene = scene
        self.buffers = SimBuffers(scene)

    # -------------------------------------------------------------- acquire
    def acquire_actor_root_state_tensor(self):
        return self.scene.root_state

    def acquire_dof_state_tensor(self):
        return self.scene.dof_state

    def acquire_rigid_body_state_tensor(self):
        return self.scene.body_state

    def acquire_net_contact_force_tensor(self):
        return self.scene.net_contact

    def acquire_force_sensor_tensor(self):
        return self.scene.sensor_forces

    def acquire_dof_force_tensor(self):
        return self.scene.dof_force

    # -------------------------------------------------------------- refresh
    def refresh_actor_root_state_tensor(self):
        """Repack root/body/dof tensors from the canonical state (needed only
        after writing `scene.body_q` directly; every step refreshes them)."""
        self.scene.refresh_buffers()

    refresh_dof_state_tensor = refresh_actor_root_state_tensor
    refresh_rigid_body_state_tensor = refresh_actor_root_state_tensor

    def refresh_net_contact_force_tensor(self):
        pass  # written by every step (physics.py:1047-1062)

    refresh_force_sensor_tensor = refresh_net_contact_force_tensor
    refresh_dof_force_tensor = refresh_net_contact_force_tensor

    # -------------------------------------------------------------- controls
    def _copy(self, dst, src):
        src = torch.as_tensor(src, device=dst.device, dtype=dst.dtype)
        if not bool(torch.isfinite(src).all()):
            from .buffers import NonFiniteWrite
            raise NonFiniteWrite("non-finite control values")
        dst.copy_(src.reshape(dst.shape))

    def set_dof_actuation_force_tensor(self, forces):
        self._copy(self.scene.ctrl_dof_force, forces)

    def set_dof_position_target_tensor(self, targets):
        self._copy(self.scene.ctrl_dof_pos_target, targets)

    def set_dof_velocity_target_tensor(self, targets):
        self._copy(self.scene.ctrl_dof_vel_target, targets)

    def apply_rigid_body_force_tensors(self, forces=None, torques=None):
        if forces is not None:
            self._copy(self.scene.ctrl_body_force, forces)
        if torques is not None:
            self._copy(self.scene.ctrl_body_torque, torques)

    # -------------------------------------------------------------- state
    def set_actor_root_state_tensor(self, root):
        self.buffers.set_root_state(root)

    def set_actor_root_state_tensor_indexed(self, root, actor_indices):
        self.buffers.set_root_state(root, actor_indices)

    def set_dof_state_tensor(self, dof):
        self.buffers.set_dof_state(dof)

    def set_dof_state_tensor_indexed(self, dof, actor_indices):
        self.buffers.set_dof_state(dof, actor_indices)

    # -------------------------------------------------------------- stepping
    def simulate(self, n_substeps: int = 1):
        """Launch `n_substeps` fused physics steps on the scene's stream."""
        self.scene.step(n_substeps)

    def fetch_results(self, wait: bool = True):
        if wait:
            self.scene.fetch_results()
        return True
