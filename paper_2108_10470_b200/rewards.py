"""Batched reward kernels on the device (reference `pkg/src/batchsim/rewards.py`).

Same function names, parameter dataclasses and argument order as the
reference; inputs may be numpy arrays or torch tensors (moved to the
device), outputs are device tensors.  Each call is one CUDA launch
(csrc/bsim_rewards.cu, one thread per env).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


@dataclass
class LocomotionRewardParams:
    heading_weight: float = 0.5
    alive_bonus: float = 0.5
    death_penalty: float = -1.0
    termination_height: float = 0.26
    upright_threshold: float = 0.93
    upright_weight: float = 0.1
    action_cost_weight: float = 0.005
    effort_weight: float = 0.05
    dof_limit_weight: float = 0.1
    dt: float = 1 / 60


@dataclass
class AnymalRewardParams:
    w_vel_xy: float = 1.0
    w_vel_yaw: float = 0.5
    w_vel_z: float = 4.0
    w_pitch_roll: float = 0.05
    w_joint_motion: float = 0.001
    w_torque: float = 0.00002
    w_action_rate: float = 0.25
    w_collision: float = 0.001
    w_air_time: float = 2.0
    dt: float = 0.02


@dataclass
class CubeRewardParams:
    dist_reward_scale: float = -10.0
    rot_reward_scale: float = 1.0
    rot_eps: float = 0.1
    action_penalty_scale: float = -0.0002
    success_tolerance: float = 0.4
    reach_goal_bonus: float = 250.0
    fall_dist: float = 0.24
    fall_penalty: float = 0.0


@dataclass
class FrankaStackParams:
    w_stack: float = 16.0
    w_align: float = 2.0
    w_lift: float = 1.5
    w_reach: float = 0.1
    lift_height: float = 0.04
    align_tolerance: float = 0.02
    away_distance: float = 0.04


@dataclass
class TrifingerRewardParams:
    w_og: float = 1.0
    w_fo: float = 0.2
    w_fv: float = -0.05
    kernel_a: float = 50.0
    kernel_b: float = 2.0
    fingertip_term_cutoff: int = int(5e7)


def _struct(p):
    fields = [(k, C.c_double) for k in p.__dataclass_fields__]
    S = type("P", (C.Structure,), {"_fields_": fields})
    return S(*(float(getattr(p, k)) for k in p.__dataclass_fields__))


class _Args:
    """Converts inputs to contiguous device tensors of one dtype (kept alive)."""

    def __init__(self, dtype=None, device="cuda"):
        self.keep, self.dtype, self.device = [], dtype, device

    def __call__(self, x, shape=None):
        if x is None:
            return None
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float64))
        if self.dtype is None:
            self.dtype = t.dtype if t.dtype in (torch.float32, torch.float64) else torch.float32
        t = t.to(self.device, self.dtype).contiguous()
        if shape is not None:
            t = t.reshape(shape)
        self.keep.append(t)
        return t

    @property
    def fp64(self):
        return int(self.dtype == torch.float64)


def _check(rc, what):
    if rc != 0:
        raise N.NativeError(f"{what} failed ({rc})")


def _stream():
    return torch.cuda.current_stream().cuda_stream


def locomotion_reward(torso_pos, target_pos, up_proj, heading_proj, actions, dof_pos, dof_vel,
                      dof_lower, dof_upper, motor_strength, prev_potential, params):
    """(reward, potential) -- rewards.py:78-112."""
    a = _Args()
    torso = a(torso_pos)
    n = torso.shape[0]
    act = a(actions)
    D = act.shape[1]
    args = [torso, a(target_pos), a(up_proj), a(heading_proj), act, a(dof_pos), a(dof_vel),
            a(dof_lower), a(dof_upper), a(motor_strength), a(prev_potential)]
    rew = torch.empty(n, dtype=a.dtype, device=torso.device)
    pot = torch.empty(n, dtype=a.dtype, device=torso.device)
    p = _struct(params)
    _check(N.lib().bsim_reward_locomotion(n, D, a.fp64, *(t.data_ptr() for t in args), C.byref(p),
                                          rew.data_ptr(), pot.data_ptr(), _stream()), "locomotion_reward")
    return rew, pot


def anymal_reward(base_lin_vel, base_ang_vel, commands, dof_vel, dof_acc, torques, action_rate,
                  collisions, feet_air_time, params, variant="flat"):
    """rewards.py:129-158."""
    if variant not in ("flat", "rough"):
        raise ValueError(f"unknown variant {variant!r}")
    a = _Args()
    lin = a(base_lin_vel)
    n = lin.shape[0]
    tq = a(torques)
    D = tq.shape[1]
    rough = variant == "rough"
    qv = a(dof_vel) if rough else tq
    qa = a(dof_acc) if rough else tq
    ar = a(action_rate) if rough else tq
    co = a(collisions) if rough else lin
    air = a(feet_air_time) if rough else tq
    A = ar.shape[1] if rough else 0
    F = air.shape[1] if rough else 0
    out = torch.empty(n, dtype=a.dtype, device=lin.device)
    p = _struct(params)
    _check(N.lib().bsim_reward_anymal(n, D, A, F, a.fp64, lin.data_ptr(), a(base_ang_vel).data_ptr(),
                                      a(commands).data_ptr(), qv.data_ptr(), qa.data_ptr(), tq.data_ptr(),
                                      ar.data_ptr(), co.data_ptr(), air.data_ptr(), C.byref(p), int(rough),
                                      out.data_ptr(), _stream()), "anymal_reward")
    return out


def cube_reorientation_reward(object_pos, object_quat, target_pos, target_quat, actions, params):
    """(reward, goal_reset, success) -- rewards.py:161-176."""
    a = _Args()
    op = a(object_pos)
    n = op.shape[0]
    act = a(actions)
    out = torch.empty(n, dtype=a.dtype, device=op.device)
    reset = torch.empty(n, dtype=torch.uint8, device=op.device)
    succ = torch.empty(n, dtype=torch.uint8, device=op.device)
    p = _struct(params)
    _check(N.lib().bsim_reward_cube(n, act.shape[1], a.fp64, op.data_ptr(), a(object_quat).data_ptr(),
                                    a(target_pos).data_ptr(), a(target_quat).data_ptr(), act.data_ptr(),
                                    C.byref(p), out.data_ptr(), reset.data_ptr(), succ.data_ptr(), _stream()),
           "cube_reorientation_reward")
    return out, reset.bool(), succ.bool()


def franka_stack_reward(cubeA_pos, cubeB_pos, gripper_pos, lfinger_pos, rfinger_pos, params):
    """rewards.py:200-219."""
    a = _Args()
    ca = a(cubeA_pos)
    n = ca.shape[0]
    out = torch.empty(n, dtype=a.dtype, device=ca.device)
    p = _struct(params)
    _check(N.lib().bsim_reward_franka(n, a.fp64, ca.data_ptr(), a(cubeB_pos).data_ptr(), a(gripper_pos).data_ptr(),
                                      a(lfinger_pos).data_ptr(), a(rfinger_pos).data_ptr(), C.byref(p),
                                      out.data_ptr(), _stream()), "franka_stack_reward")
    return out


def trifinger_reward(cube_pos, prev_cube_pos, cube_quat, target_pos, target_quat, fingertip_pos,
                     prev_fingertip_pos, fingertip_vel, timestep, params):
    """rewards.py:179-197; fingertip arrays are (n, F, 3), timestep (n,) integer steps."""
    a = _Args()
    cp = a(cube_pos)
    n = cp.shape[0]
    ft = a(fingertip_pos)
    F = ft.shape[1] if ft.dim() == 3 else 0
    ts = timestep if isinstance(timestep, torch.Tensor) else torch.as_tensor(np.asarray(timestep))
    ts = torch.broadcast_to(ts.to(cp.device, torch.int64), (n,)).contiguous()
    a.keep.append(ts)
    args = [cp, a(prev_cube_pos), a(cube_quat), a(target_pos), a(target_quat), ft, a(prev_fingertip_pos),
            a(fingertip_vel)]
    out = torch.empty(n, dtype=a.dtype, device=cp.device)
    p = _struct(params)
    _check(N.lib().bsim_reward_trifinger(n, F, a.fp64, *(t.data_ptr() for t in args), ts.data_ptr(), C.byref(p),
                                         out.data_ptr(), _stream()), "trifinger_reward")
    return out


def ingenuity_reward(pos, target, local_up_z, spin_rate):
    """rewards.py:115-121: R_pos * (1 + R_upright + R_spin)."""
    a = _Args()
    ps = a(pos)
    n = ps.shape[0]
    spin = a(spin_rate)
    spin = spin.reshape(n, -1)
    out = torch.empty(n, dtype=a.dtype, device=ps.device)
    _check(N.lib().bsim_reward_ingenuity(n, spin.shape[1], a.fp64, ps.data_ptr(), a(target).data_ptr(),
                                         a(local_up_z).data_ptr(), spin.data_ptr(), out.data_ptr(), _stream()),
           "ingenuity_reward")
    return out


def amp_imitation_reward(d_score):
    """rewards.py:222-225: -ln(1 - clip(D, 1e-4, 1 - 1e-4)), same shape as d_score."""
    a = _Args()
    d = a(d_score)
    out = torch.empty_like(d)
    _check(N.lib().bsim_reward_amp(d.numel(), a.fp64, d.data_ptr(), out.data_ptr(), _stream()),
           "amp_imitation_reward")
    return out
