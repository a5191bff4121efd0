"""Host-side packing: SceneLayout -> the flat arrays behind bsim_layout_t /
bsim_state_t (include/batchsim_b200.h).

Used once at scene construction; the Scene uploads the results to HBM.
"""

from __future__ import annotations

import ctypes as C

import os

import numpy as np

from . import _native as N
from .layout import SceneLayout
from .params import SimParams


def pack_tables(L: SceneLayout, fp64: bool = False):
    """Static tables as numpy arrays (int32 / raw struct bytes) for the float or
    double struct variants."""
    J = L.joints_per_env
    joints = ((N.Joint64 if fp64 else N.Joint) * max(J, 1))()
    for i, j in enumerate(L.joints):
        r = joints[i]
        r.kind, r.parent, r.child, r.dof, r.actor, r.has_limits = (
            j.kind, j.parent, j.child, j.dof, j.actor, int(j.has_limits))
        for k in range(3):
            r.axis[k], r.origin_pos[k], r.child_pos[k] = j.axis[k], j.origin_pos[k], j.child_pos[k]
        for k in range(4):
            r.origin_quat[k], r.child_quat[k] = j.origin_quat[k], j.child_quat[k]
    T = L.tendons_per_env
    tendons = ((N.Tendon64 if fp64 else N.Tendon) * max(T, 1))()
    flat_paths, path_off = [], []
    for t in range(T):
        paths = L.spatial_paths[t]
        if paths:
            path_off.append(len(flat_paths))
            flat_paths.append(len(paths))
            for p in paths:
                flat_paths += [len(p)] + list(p)
        else:
            path_off.append(0)
    for t in range(T):
        r = tendons[t]
        ti, tf = L.tendon_int[t], L.tendon_flt[t]
        r.kind, r.first, r.count, r.has_limits, r.reaction_body, r.actor = (int(x) for x in ti[:6])
        r.path_offset = path_off[t]
        (r.rest_length, r.stiffness, r.damping, r.limit_lo, r.limit_hi,
         r.limit_stiffness) = (float(x) for x in tf[:6])
    n_el = len(L.telem_int)
    elems = ((N.TendonElem64 if fp64 else N.TendonElem) * max(n_el, 1))()
    for i in range(n_el):
        r = elems[i]
        r.index, r.parent, r.joint = (int(x) for x in L.telem_int[i, :3])
        for k in range(4):
            r.v[k] = float(L.telem_flt[i, k])
    as_bytes = lambda arr: np.frombuffer(bytes(arr), dtype=np.uint8).copy()  # noqa: E731
    return {
        "joints": as_bytes(joints),
        "plane_body": np.ascontiguousarray(L.plane_body, np.int32).reshape(-1) if L.planes_per_env else np.zeros(1, np.int32),
        "pair_body": np.ascontiguousarray(L.pair_body, np.int32).reshape(-1) if L.pairs_per_env else np.zeros(2, np.int32),
        "sensor_body": np.ascontiguousarray(L.sensor_body, np.int32) if L.sensors_per_env else np.zeros(1, np.int32),
        "actor_body_offset": np.array(L.actor_body_offset + [L.bodies_per_env], np.int32),
        "actor_dof_offset": np.array(L.actor_dof_offset + [L.dofs_per_env], np.int32),
        "tendons": as_bytes(tendons),
        "tendon_elems": as_bytes(elems),
        "spatial_paths": np.array(flat_paths or [0], np.int32),
        "pair_kind": np.ascontiguousarray(L.pair_kind, np.int32) if L.pairs_per_env else np.zeros(1, np.int32),
        "pair_ext": (np.ascontiguousarray(L.pair_ext, np.float64 if fp64 else np.float32).reshape(-1)
                     if L.pairs_per_env else np.zeros(4, np.float64 if fp64 else np.float32)),
        "sweep_sched": sched_table(L),
    }


def sched_table(L: SceneLayout):
    """[stages][width] int32 row ids of SceneLayout.sweep_schedule, -1 padded."""
    _, stages, width = L.sweep_schedule()
    t = np.full((max(len(stages), 1), max(width, 1)), -1, np.int32)
    for k, st in enumerate(stages):
        t[k, :len(st)] = st
    return t.reshape(-1)


def init_state_arrays(L: SceneLayout, E: int, params: SimParams, env_origins: np.ndarray,
                      fp64: bool = False):
    """Real (float32 or float64) / int8 / bool state arrays in the reference
    shapes (env-local poses)."""
    B, D, J, P, Q = (L.bodies_per_env, L.dofs_per_env, L.joints_per_env, L.planes_per_env,
                     L.pairs_per_env)
    A, S = L.actors_per_env, L.sensors_per_env
    f32 = np.float64 if fp64 else np.float32
    body_q = np.zeros((E * B, 13), f32)
    body_q[:, 6] = 1.0
    jp = L.joint_param_defaults()
    a = {
        "body_q": body_q,
        "friction_anchor": np.full((P, E, 3), np.nan, f32),
        "nonfinite": np.zeros(E, np.bool_),
        "env_origins": np.ascontiguousarray(env_origins, f32),
        "inv_mass": np.tile(L.inv_mass, E).astype(f32),
        "inertia_local": np.tile(L.inertia, (E, 1)).astype(f32),
        "inv_inertia_local": np.tile(L.inv_inertia, (E, 1)).astype(f32),
        "gravity": np.tile(np.asarray(params.gravity, float), (E, 1)).astype(f32),
        "mu_static": np.full(E, params.static_friction, f32),
        "mu_dynamic": np.full(E, params.dynamic_friction, f32),
        "joint_stiffness": np.repeat(jp[0][:, None], E, 1).astype(f32),
        "joint_damping": np.repeat(jp[1][:, None], E, 1).astype(f32),
        "joint_armature": np.repeat(jp[2][:, None], E, 1).astype(f32),
        "joint_friction": np.repeat(jp[3][:, None], E, 1).astype(f32),
        "joint_limit_lo": np.repeat(jp[4][:, None], E, 1).astype(f32),
        "joint_limit_hi": np.repeat(jp[5][:, None], E, 1).astype(f32),
        "plane_off": np.repeat(L.plane_off.reshape(P, 1, 3), E, 1).astype(f32),
        "plane_rad": np.repeat(L.plane_rad.reshape(P, 1), E, 1).astype(f32),
        "pair_off": np.repeat(L.pair_off.reshape(Q, 1, 2, 3), E, 1).astype(f32),
        "pair_rad": np.repeat(L.pair_rad.reshape(Q, 1, 2), E, 1).astype(f32),
        "ctrl_dof_force": np.zeros(E * D, f32),
        "ctrl_dof_pos_target": np.zeros(E * D, f32),
        "ctrl_dof_vel_target": np.zeros(E * D, f32),
        "ctrl_body_force": np.zeros((E * B, 3), f32),
        "ctrl_body_torque": np.zeros((E * B, 3), f32),
        "dof_mode": np.tile(L.dof_mode, E).astype(np.int8),
        "root_state": np.zeros((E * A, 13), f32),
        "body_state": np.zeros((E * B, 13), f32),
        "dof_state": np.zeros((E * D, 2), f32),
        "net_contact": np.zeros((E * B, 3), f32),
        "dof_force": np.zeros(E * D, f32),
        "sensor_forces": np.zeros((E * S, 6), f32),
    }
    return a


def layout_struct(L: SceneLayout, E: int, ptrs: dict, env_offset: int = 0,
                  topology_id: int = 0) -> N.Layout:
    s = N.Layout()
    s.topology_id = topology_id
    (s.num_envs, s.actors_per_env, s.bodies_per_env, s.dofs_per_env, s.joints_per_env,
     s.planes_per_env, s.pairs_per_env, s.sensors_per_env, s.tendons_per_env, s.env_offset) = (
        E, L.actors_per_env, L.bodies_per_env, L.dofs_per_env, L.joints_per_env,
        L.planes_per_env, L.pairs_per_env, L.sensors_per_env, L.tendons_per_env, env_offset)
    mode, stages, width = L.sweep_schedule()
    s.sched_stages, s.sched_width = len(stages), width        # 0 stages: the one-lane sequential sweep
    s.sched_flags = 1 if mode == "joints" else 0
    if os.environ.get("BSIM_NO_SCHED"):          # timing experiment
        s.sched_stages = 0
    for name in N.LAYOUT_PTRS:
        setattr(s, name, C.c_void_p(ptrs[name]))
    return s


def params_struct(p: SimParams, fp64: bool = False):
    return (N.Params64 if fp64 else N.Params)(p.dt, p.position_iterations, p.velocity_iterations, p.max_bias, p.restitution,
                    p.bounce_threshold, p.rest_offset, p.friction_offset_threshold,
                    p.solver_offset_slop, p.max_force, p.linear_damping, p.angular_damping,
                    p.max_linear_velocity, p.max_angular_velocity)


def state_struct(ptrs: dict) -> N.State:
    s = N.State()
    for name in N.STATE_PTRS:
        setattr(s, name, C.c_void_p(ptrs[name]))
    return s
