"""Generate golden vectors by running the REFERENCE implementation.

Run here (the reference is importable from /root/reference; it does not
exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each physics case builds a reference `batchsim.physics.Scene`
(/root/reference/pkg/src/batchsim/physics.py:143), perturbs it, then records
the full canonical state before and after every `Scene.step()` so tests can
replay the steps one at a time (teacher forcing) against the oracle and the
CUDA path.  All arrays are float64 exactly as the reference produced them.
Env-layer, reward and buffer-API cases are recorded the same way.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from batchsim import models as RM  # noqa: E402
from batchsim import rewards as RR  # noqa: E402
from batchsim.buffers import SimBuffers  # noqa: E402
from batchsim.envs import make_env  # noqa: E402
from batchsim.model import load_model  # noqa: E402
from batchsim.physics import MODE_VELOCITY, Scene, SimParams  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

STATE = ("pos", "quat", "linvel", "angvel", "_friction_anchor", "nonfinite", "dof_state",
         "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
         "ctrl_body_torque", "dof_mode")
PARAMS = ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static",
          "mu_dynamic", "joint_stiffness", "joint_damping", "joint_armature", "joint_friction",
          "joint_limit_lo", "joint_limit_hi", "plane_off", "plane_rad", "pair_off", "pair_rad",
          "env_origins")
OUTPUTS = ("root_state", "body_state", "dof_state", "net_contact", "dof_force",
           "sensor_forces", "nonfinite")


# ---------------------------------------------------------------- models
def kitchen_sink_docs():
    """Authored multi-actor scene exercising every joint kind, capsule/box
    slots, sphere-sphere pairs, armature, dry friction, velocity drives and
    fixed + spatial tendons (paths no reference test pins)."""
    arm = {
        "name": "arm", "fixed_base": True,
        "links": [
            {"name": "base", "mass": 2.0, "inertia": [0.1, 0.1, 0.1],
             "shape": {"kind": "box", "params": [0.1, 0.1, 0.05]}},
            {"name": "l1", "mass": 0.5, "inertia": [0.01, 0.01, 0.004],
             "shape": {"kind": "capsule", "params": [0.04, 0.1]}, "collision": True},
            {"name": "l2", "mass": 0.4, "inertia": [0.008, 0.008, 0.003], "collision": False},
            {"name": "l3", "mass": 0.3, "inertia": [0.004, 0.005, 0.002],
             "shape": {"kind": "capsule", "params": [0.03, 0.08], "offset": [0, 0, -0.08]}},
            {"name": "tip", "mass": 0.2, "inertia": [0.002, 0.002, 0.002],
             "shape": {"kind": "sphere", "params": [0.06]}},
        ],
        "joints": [
            {"name": "j_rev", "kind": "revolute", "parent": "base", "child": "l1",
             "axis": [0, 1, 0.2], "limits": [-0.8, 0.8], "origin": {"pos": [0, 0, 0.3]},
             "child_origin": {"pos": [0, 0, -0.1]}, "stiffness": 30.0, "damping": 2.0,
             "armature": 0.02, "friction": 0.3},
            {"name": "j_pri", "kind": "prismatic", "parent": "l1", "child": "l2",
             "axis": [1, 0, 0], "limits": [-0.1, 0.15], "origin": {"pos": [0, 0, 0.12]},
             "damping": 5.0},
            {"name": "j_sph", "kind": "spherical", "parent": "l2", "child": "l3",
             "origin": {"pos": [0.05, 0, 0.05], "quat": [0, 0.2588190451, 0, 0.9659258263]}},
            {"name": "j_fix", "kind": "fixed", "parent": "l3", "child": "tip",
             "origin": {"pos": [0, 0, -0.18]}},
        ],
        "tendons": [
            {"name": "couple", "kind": "fixed", "stiffness": 4.0, "damping": 0.3,
             "rest_length": 0.05, "limits": [-0.2, 0.2], "limit_stiffness": 10.0,
             "joints": [{"dof": "j_rev", "coefficient": 1.0},
                        {"dof": "j_pri", "coefficient": -0.5, "parent": 0}]},
            {"name": "string", "kind": "spatial", "stiffness": 20.0, "damping": 0.5,
             "rest_length": 0.3,
             "attachments": [{"link": "base", "offset": [0.05, 0, 0.05]},
                             {"link": "l1", "offset": [0.03, 0, 0.0], "parent": 0},
                             {"link": "l3", "offset": [0, 0.02, -0.1], "parent": 1,
                              "weight": 0.8},
                             {"link": "tip", "offset": [0, -0.03, 0], "parent": 1}]},
        ],
        "sensors": ["l1", "tip"],
    }
    ball = {"name": "ball", "links": [
        {"name": "ball", "mass": 0.5, "inertia": [0.002, 0.002, 0.002],
         "shape": {"kind": "sphere", "params": [0.07]}}]}
    box = {"name": "crate", "links": [
        {"name": "crate", "mass": 1.0, "inertia": [0.007, 0.005, 0.004],
         "shape": {"kind": "box", "params": [0.08, 0.06, 0.05]}}]}
    return [arm, ball, box]


# ---------------------------------------------------------------- helpers
def snapshot(s, names):
    return {k: np.array(getattr(s, k), copy=True) for k in names}


def record_steps(s, steps, control_fn, pre_step=None):
    """[t] inputs (state before step t), [t] outputs (after step t)."""
    ins = {k: [] for k in STATE}
    outs = {k: [] for k in OUTPUTS + ("pos", "quat", "linvel", "angvel", "_friction_anchor")}
    for t in range(steps):
        control_fn(s, t)
        if pre_step is not None:
            pre_step(s, t)
        for k, v in snapshot(s, STATE).items():
            ins[k].append(v)
        s.step()
        for k, v in snapshot(s, outs).items():
            outs[k].append(v)
    return ({f"in_{k}": np.stack(v) for k, v in ins.items()},
            {f"out_{k}": np.stack(v) for k, v in outs.items()})


def save(name, meta, arrays):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, meta=np.array(json.dumps(meta)), **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.0f} KiB")


def params_meta(p):
    d = dict(p.__dict__)
    d["gravity"] = list(d["gravity"])
    return d


def physics_case(name, models_spec, E, params, steps, setup, control_fn, spacing=4.0,
                 ground=True, pre_step=None, warmup=0):
    """models_spec: list of registry names or JSON documents."""
    models = [getattr(RM, m)() if isinstance(m, str) else load_model(m) for m in models_spec]
    s = Scene(models, E, params, spacing=spacing, ground=ground)
    setup(s)
    for t in range(warmup):
        control_fn(s, -1 - t)
        s.step()
    ins, outs = record_steps(s, steps, control_fn, pre_step)
    meta = {"kind": "physics", "models": models_spec, "num_envs": E, "steps": steps,
            "params": params_meta(params), "spacing": spacing, "ground": ground}
    arrays = {**ins, **outs, **{f"param_{k}": np.array(getattr(s, k)) for k in PARAMS}}
    # collide(): the reference contact list at the final state (physics.py:500-517)
    cl = s.collide()
    arrays["collide_body_a"] = np.array([c.body_a for c in cl], np.int64)
    arrays["collide_body_b"] = np.array([c.body_b for c in cl], np.int64)
    arrays["collide_depth"] = np.array([c.depth for c in cl], float)
    arrays["collide_point"] = np.array([c.point for c in cl], float).reshape(-1, 3)
    arrays["collide_normal"] = np.array([c.normal for c in cl], float).reshape(-1, 3)
    arrays["collide_has_anchor"] = np.array([c.friction_anchor is not None for c in cl], bool)
    arrays["final_pos"] = s.pos.copy()
    arrays["final_quat"] = s.quat.copy()
    save(name, meta, arrays)


def rng_targets(scale, seed):
    rng = np.random.default_rng(seed)

    def fn(s, t):
        s.ctrl_dof_pos_target[:] = rng.uniform(-scale, scale, s.num_dofs)
    return fn


def reset_walkers(height, yaw=0.1, qscale=0.1, vscale=0.0, seed=1):
    def fn(s):
        rng = np.random.default_rng(seed)
        buf = SimBuffers(s)
        root = s.root_state.copy()
        E = s.num_envs
        yaw_ = rng.uniform(-yaw, yaw, E)
        root[:, 0:3] = s.env_origins + [0, 0, height]
        root[:, 3:7] = np.stack([np.zeros(E), np.zeros(E), np.sin(yaw_ / 2), np.cos(yaw_ / 2)], -1)
        root[:, 7:13] = rng.uniform(-vscale, vscale, (E, 6))
        buf.set_root_state(root)
        dof = s.dof_state.copy()
        dof[:, 0] = rng.uniform(-qscale, qscale, s.num_dofs)
        dof[:, 1] = rng.uniform(-vscale, vscale, s.num_dofs)
        buf.set_dof_state(dof)
    return fn


# ---------------------------------------------------------------- cases
def main():
    dt = 1.0 / 120.0
    # Ant analog: settle onto the ground then walk with random targets.
    physics_case("quadruped_walk", ["quadruped"], 12, SimParams(dt=dt), 8,
                 reset_walkers(0.37, vscale=0.3), rng_targets(0.6, 11), warmup=30)
    # ANYmal analog.
    physics_case("quadruped12_walk", ["quadruped12"], 8, SimParams(dt=dt), 6,
                 reset_walkers(0.34, vscale=0.3), rng_targets(0.5, 12), warmup=30)
    # Falling / landing (restitution, bounce threshold, fresh anchors).
    physics_case("quadruped_drop", ["quadruped"], 8, SimParams(dt=dt, restitution=0.5), 12,
                 reset_walkers(0.6, yaw=1.0, qscale=0.8, vscale=2.0, seed=5),
                 rng_targets(0.6, 13))

    def pend_setup(s):
        buf = SimBuffers(s)
        dof = s.dof_state.copy()
        dof[:, 0] = np.linspace(0.3, np.pi / 2, s.num_dofs)
        buf.set_dof_state(dof)
    physics_case("pendulum_swing", ["pendulum"], 3, SimParams(dt=1 / 200), 12, pend_setup,
                 lambda s, t: None, ground=False, warmup=20)

    def chain_setup(s):
        buf = SimBuffers(s)
        dof = s.dof_state.copy()
        dof[:, 0] = 0.5
        dof[:, 1] = np.linspace(-1, 1, s.num_dofs)
        buf.set_dof_state(dof)
    physics_case("chain3_free", ["chain3"], 2, SimParams(dt=dt), 12, chain_setup,
                 lambda s, t: None, ground=False)

    def cart_setup(s):
        buf = SimBuffers(s)
        dof = s.dof_state.copy()
        rng = np.random.default_rng(3)
        dof[:, 0] = rng.uniform(-0.5, 0.5, s.num_dofs)
        dof[:, 1] = rng.uniform(-1, 1, s.num_dofs)
        dof[0::2, 0] = [3.95, -3.9, 0.0, 1.0][: s.num_envs]  # near the slider limits
        buf.set_dof_state(dof)
    frng = np.random.default_rng(4)

    def cart_force(s, t):
        f = np.zeros(s.num_dofs)
        f[0::2] = frng.uniform(-10, 10, s.num_envs)
        s.ctrl_dof_force[:] = f
    physics_case("cartpole_force", ["cartpole"], 4, SimParams(dt=dt), 12, cart_setup, cart_force,
                 ground=False)

    def sphere_setup(s):
        r = 0.1
        for e in range(s.num_envs):
            s.pos[e] = s.env_origins[e] + [0, 0, r + 0.02 * e]
            s.linvel[e] = [0.3 * e, -0.2, -2.0 + 0.5 * e]
            s.angvel[e] = [0.5, -1.0 * e, 0.2]
    physics_case("sphere_bounce", ["free_sphere"], 4, SimParams(dt=1 / 240, restitution=0.8),
                 16, sphere_setup, lambda s, t: None)

    th = np.arctan(0.6) - np.radians(3)

    def box_setup(s):
        for e in range(s.num_envs):
            s.pos[e] = s.env_origins[e] + [0, 0, 0.1 - 0.002 * e]
            s.angvel[e] = [0.0, 0.0, 0.5 * e]
    physics_case("box_incline", ["free_box"], 3,
                 SimParams(dt=1 / 240, gravity=(9.81 * np.sin(th), 0.0, -9.81 * np.cos(th)),
                           static_friction=0.6, dynamic_friction=0.5),
                 10, box_setup, lambda s, t: None, warmup=40)

    # Authored multi-actor scene.
    docs = kitchen_sink_docs()

    def ks_setup(s):
        buf = SimBuffers(s)
        root = s.root_state.copy()
        E, A = s.num_envs, s.actors_per_env
        rng = np.random.default_rng(7)
        for e in range(E):
            o = s.env_origins[e]
            root[e * A + 0, 0:3] = o + [0, 0, 0.05]
            root[e * A + 1, 0:3] = o + [0.25 + 0.02 * e, 0.0, 0.5]
            root[e * A + 1, 7:10] = [-0.5, 0.0, -0.5]
            root[e * A + 2, 0:3] = o + [-0.4, 0.1, 0.06]
            q = rng.normal(size=4) * [0.1, 0.1, 0.5, 0] + [0, 0, 0, 1]
            root[e * A + 2, 3:7] = q / np.linalg.norm(q)
            root[e * A + 2, 10:13] = [0.0, 0.0, 2.0]
        buf.set_root_state(root)
        dof = s.dof_state.copy()
        dof[:, 0] = rng.uniform(-0.3, 0.3, s.num_dofs)
        dof[:, 1] = rng.uniform(-0.5, 0.5, s.num_dofs)
        buf.set_dof_state(dof)
        # prismatic joint driven in velocity mode; revolute position mode
        D = s.dofs_per_env
        s.dof_mode[1::D] = MODE_VELOCITY
        s.joint_damping[1, :] = 5.0
    krng = np.random.default_rng(8)

    def ks_ctrl(s, t):
        D, B = s.dofs_per_env, s.bodies_per_env
        s.ctrl_dof_pos_target[0::D] = krng.uniform(-0.5, 0.5, s.num_envs)
        s.ctrl_dof_vel_target[1::D] = krng.uniform(-0.3, 0.3, s.num_envs)
        f = np.zeros((s.num_bodies, 3))
        f[B - 1::B] = krng.uniform(-3, 3, (s.num_envs, 3))
        s.ctrl_body_force[:] = f
        tq = np.zeros((s.num_bodies, 3))
        tq[B - 1::B] = krng.uniform(-0.2, 0.2, (s.num_envs, 3))
        s.ctrl_body_torque[:] = tq
    physics_case("kitchen_sink", docs, 3,
                 SimParams(dt=dt, linear_damping=0.05, angular_damping=0.1, restitution=0.3),
                 10, ks_setup, ks_ctrl, warmup=10)

    # NaN containment: poison env 1 mid-run (tests/test_physics.py:242-258).
    def nan_pre(s, t):
        if t == 2:
            s.linvel[s.bodies_per_env + 1, 0] = np.nan
    physics_case("quadruped_nan", ["quadruped"], 3, SimParams(dt=dt), 5,
                 reset_walkers(0.37), rng_targets(0.3, 21), pre_step=nan_pre)

    env_cases()
    buffer_cases()
    reward_cases()
    reward_extra_cases()
    randomize_cases()


# ------------------------------------------------------------- env layer
ENV_STATE = ("episode_steps", "reset_count", "actions")


def env_cases():
    """EnvBatch.step traces (envs.py:178-200) for the two locomotion tasks.
    Records obs/reward/done and the reset rows the reference drew."""
    for task, E, steps in (("quadruped", 8, 30), ("quadruped-anymal-obs", 8, 24)):
        env = make_env(task, num_envs=E, seed=3, episode_length=25)
        rng = np.random.default_rng(99)
        rec = {k: [] for k in ("actions", "obs", "reward", "done", "timeout", "root_state",
                               "dof_state", "pos", "quat", "linvel", "angvel",
                               "_friction_anchor", "sensor_forces", "dof_force",
                               "ctrl_dof_pos_target", "episode_steps", "reset_count",
                               "extra_before", "extra_after")}
        obs0 = env.reset()
        extra_name = "potentials" if task == "quadruped" else "commands"
        for t in range(steps):
            a = rng.uniform(-1.2, 1.2, (E, env.act_dim))
            if t == 5:
                # knock env 2 over so the termination path fires
                root = env.scene.root_state.copy()
                root[2, 2] = 0.1
                env.buffers.set_root_state(root, [2])
            rec["extra_before"].append(np.array(getattr(env, extra_name), copy=True))
            pre = snapshot(env.scene, ("pos", "quat", "linvel", "angvel", "_friction_anchor",
                                       "root_state", "dof_state", "sensor_forces", "dof_force"))
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
            rec["extra_after"].append(np.array(getattr(env, extra_name), copy=True))
        arrays = {k: np.stack(v) for k, v in rec.items()}
        arrays["obs0"] = obs0
        arrays["final_pos"] = env.scene.pos.copy()
        arrays["final_quat"] = env.scene.quat.copy()
        arrays["final_linvel"] = env.scene.linvel.copy()
        arrays["final_angvel"] = env.scene.angvel.copy()
        arrays["final_dof_state"] = env.scene.dof_state.copy()
        arrays["env_origins"] = env.scene.env_origins.copy()
        meta = {"kind": "env", "task": task, "num_envs": E, "steps": steps, "seed": 3,
                "episode_length": 25}
        save(f"env_{task.replace('-', '_')}", meta, arrays)


def buffer_cases():
    """SimBuffers indexed setters (buffers.py:127-178): state after a root
    teleport and a DOF write on a subset of actors, incl. forward kinematics."""
    s = Scene([RM.quadruped()], 6, SimParams(dt=1 / 120))
    rng = np.random.default_rng(5)
    for _ in range(8):
        s.ctrl_dof_pos_target[:] = rng.uniform(-0.4, 0.4, s.num_dofs)
        s.step()
    buf = SimBuffers(s)
    before = snapshot(s, ("pos", "quat", "linvel", "angvel", "root_state", "body_state", "dof_state"))
    root = s.root_state.copy()
    idx_r = np.array([4, 1])
    root[idx_r, 0:3] = s.env_origins[idx_r] + rng.uniform([-1, -1, 0.3], [1, 1, 0.6], (2, 3))
    q = rng.normal(size=(2, 4))
    root[idx_r, 3:7] = q * 1.7  # non-unit: the setter renormalises
    root[idx_r, 7:13] = rng.uniform(-0.5, 0.5, (2, 6))
    buf.set_root_state(root, idx_r)
    mid = snapshot(s, ("pos", "quat", "linvel", "angvel", "root_state", "body_state", "dof_state"))
    dof = s.dof_state.copy()
    idx_d = np.array([0, 3, 5])
    view = dof.reshape(6, -1, 2)
    view[idx_d] = rng.uniform(-0.6, 0.6, view[idx_d].shape)
    buf.set_dof_state(dof, idx_d)
    after = snapshot(s, ("pos", "quat", "linvel", "angvel", "root_state", "body_state", "dof_state"))
    arrays = {**{f"before_{k}": v for k, v in before.items()},
              **{f"mid_{k}": v for k, v in mid.items()},
              **{f"after_{k}": v for k, v in after.items()},
              "root_values": root, "dof_values": dof, "idx_root": idx_r, "idx_dof": idx_d,
              "env_origins": s.env_origins}
    save("buffers_quadruped", {"kind": "buffers", "num_envs": 6}, arrays)


def randomize_cases():
    """DomainRandomizer (randomize.py:86-189) on an Ant-analog scene, and a
    randomised + correlated-obs-noise env trace (uncorrelated noise off: the
    reference draws it from one batch-wide sequential stream)."""
    from batchsim.randomize import DEFAULT_SCHEDULE, DomainRandomizer
    watched = ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static", "mu_dynamic",
               "joint_stiffness", "joint_damping", "joint_limit_lo", "joint_limit_hi", "plane_rad",
               "plane_off")
    s = Scene([RM.quadruped()], 6, SimParams(dt=1 / 120))
    dr = DomainRandomizer(s, DEFAULT_SCHEDULE, seed=11)
    arrays = {}
    dr.randomize(np.arange(6), step=0)
    arrays.update({f"e0_{k}": getattr(s, k).copy() for k in watched})
    dr.randomize(np.array([1, 3]), step=100)            # not due: unchanged
    dr.randomize(np.array([0, 2, 5]), step=800)         # epoch 1 for three envs
    arrays.update({f"e1_{k}": getattr(s, k).copy() for k in watched})
    arrays["epoch"] = dr.epoch.copy()
    save("randomize_quadruped", {"kind": "randomize", "num_envs": 6, "seed": 11}, arrays)

    env = make_env("quadruped", num_envs=6, seed=4, episode_length=12, randomize=True, obs_noise=True,
                   obs_noise_uncorr=0.0)
    rng = np.random.default_rng(5)
    rec = {k: [] for k in ("actions", "obs", "reward", "done", "gravity", "joint_stiffness", "corr")}
    obs0 = env.reset()
    for t in range(20):
        a = rng.uniform(-1, 1, (6, env.act_dim))
        out = env.step(a)
        rec["actions"].append(a)
        rec["obs"].append(out.obs.copy())
        rec["reward"].append(out.reward.copy())
        rec["done"].append(out.done.copy())
        rec["gravity"].append(env.scene.gravity.copy())
        rec["joint_stiffness"].append(env.scene.joint_stiffness.copy())
        rec["corr"].append(env._corr_noise.copy())
    arrays = {k: np.stack(v) for k, v in rec.items()}
    arrays["obs0"] = obs0
    save("env_quadruped_dr_noise", {"kind": "env", "task": "quadruped", "num_envs": 6, "steps": 20,
                                    "seed": 4, "episode_length": 12}, arrays)


def reward_cases():
    """Batched reward kernels on random inputs (rewards.py:78-219)."""
    rng = np.random.default_rng(2024)
    N, D = 512, 8
    lp = RR.LocomotionRewardParams(dt=1 / 60)
    loc = dict(torso=rng.normal(size=(N, 3)) + [0, 0, 0.3], target=rng.normal(size=(N, 3), scale=5),
               up=rng.uniform(0.5, 1.0, N), heading=rng.uniform(-1, 1, N),
               actions=rng.normal(size=(N, D)), dof_pos=rng.uniform(-1.05, 1.05, (N, D)),
               dof_vel=rng.normal(size=(N, D)), lo=np.full(D, -1.0), hi=np.full(D, 1.0),
               strength=rng.uniform(0.5, 1.0, D), prev=rng.normal(size=N, scale=10))
    r, pot = RR.locomotion_reward(loc["torso"], loc["target"], loc["up"], loc["heading"],
                                  loc["actions"], loc["dof_pos"], loc["dof_vel"], loc["lo"],
                                  loc["hi"], loc["strength"], loc["prev"], lp)
    ap = RR.AnymalRewardParams(dt=1 / 60)
    an = dict(lin=rng.normal(size=(N, 3)), ang=rng.normal(size=(N, 3)),
              cmd=rng.uniform(-1, 1, (N, 3)), torques=rng.normal(size=(N, 12), scale=20))
    ar = RR.anymal_reward(an["lin"], an["ang"], an["cmd"], None, None, an["torques"], None,
                          None, None, ap, variant="flat")
    cp = RR.CubeRewardParams()
    q1 = rng.normal(size=(N, 4)); q1 /= np.linalg.norm(q1, axis=1, keepdims=True)
    q2 = rng.normal(size=(N, 4)); q2 /= np.linalg.norm(q2, axis=1, keepdims=True)
    q2[: N // 4] = q1[: N // 4] + rng.normal(size=(N // 4, 4), scale=0.05)
    q2 /= np.linalg.norm(q2, axis=1, keepdims=True)
    cu = dict(opos=rng.normal(size=(N, 3), scale=0.1), oq=q1,
              tpos=rng.normal(size=(N, 3), scale=0.1), tq=q2, actions=rng.normal(size=(N, 20)))
    cr, creset, csucc = RR.cube_reorientation_reward(cu["opos"], cu["oq"], cu["tpos"], cu["tq"],
                                                     cu["actions"], cp)
    fp = RR.FrankaStackParams()
    fr = dict(a=rng.normal(size=(N, 3), scale=0.05) + [0, 0, 0.04],
              b=rng.normal(size=(N, 3), scale=0.05), g=rng.normal(size=(N, 3), scale=0.05),
              l=rng.normal(size=(N, 3), scale=0.05), r=rng.normal(size=(N, 3), scale=0.05))
    fr["b"][: N // 8] = fr["a"][: N // 8] + [0.001, 0.001, -0.05]
    fr["g"][: N // 8] = fr["a"][: N // 8] + [0, 0, 0.2]
    frr = RR.franka_stack_reward(fr["a"], fr["b"], fr["g"], fr["l"], fr["r"], fp)
    arrays = {**{f"loc_{k}": v for k, v in loc.items()}, "loc_reward": r, "loc_potential": pot,
              **{f"any_{k}": v for k, v in an.items()}, "any_reward": ar,
              **{f"cube_{k}": v for k, v in cu.items()}, "cube_reward": cr,
              "cube_success": csucc, **{f"franka_{k}": v for k, v in fr.items()},
              "franka_reward": frr}
    save("rewards", {"kind": "rewards", "n": N}, arrays)


def reward_extra_cases():
    """The remaining reward kernels: trifinger (rewards.py:179-197, both sides
    of the fingertip-term cutoff), ingenuity (115-121), AMP (222-225, incl.
    the clip edges) and the nine-term rough ANYmal variant (129-158)."""
    rng = np.random.default_rng(2025)
    N, F = 512, 3
    tp = RR.TrifingerRewardParams()
    q1 = rng.normal(size=(N, 4)); q1 /= np.linalg.norm(q1, axis=1, keepdims=True)
    q2 = rng.normal(size=(N, 4)); q2 /= np.linalg.norm(q2, axis=1, keepdims=True)
    q2[: N // 4] = q1[: N // 4] + rng.normal(size=(N // 4, 4), scale=0.02)
    q2 /= np.linalg.norm(q2, axis=1, keepdims=True)
    tri = dict(cube=rng.normal(size=(N, 3), scale=0.05), prev_cube=rng.normal(size=(N, 3), scale=0.05),
               cube_quat=q1, target=rng.normal(size=(N, 3), scale=0.05), target_quat=q2,
               tip=rng.normal(size=(N, F, 3), scale=0.1), prev_tip=rng.normal(size=(N, F, 3), scale=0.1),
               tip_vel=rng.normal(size=(N, F, 3)),
               timestep=np.where(rng.uniform(size=N) < 0.5, tp.fingertip_term_cutoff - 3,
                                 tp.fingertip_term_cutoff + 3).astype(np.int64))
    tri["timestep"][0] = tp.fingertip_term_cutoff
    tri["target"][: N // 8] = tri["cube"][: N // 8]
    trr = RR.trifinger_reward(tri["cube"], tri["prev_cube"], tri["cube_quat"], tri["target"],
                              tri["target_quat"], tri["tip"], tri["prev_tip"], tri["tip_vel"],
                              tri["timestep"], tp)
    ing = dict(pos=rng.normal(size=(N, 3)), target=rng.normal(size=(N, 3)),
               up=rng.uniform(-1, 1, N), spin=rng.normal(size=(N, 3)))
    igr = RR.ingenuity_reward(ing["pos"], ing["target"], ing["up"], ing["spin"])
    d = rng.uniform(-0.2, 1.2, N)
    d[:4] = [0.0, 1.0, 1e-4, 1.0 - 1e-4]
    amr = RR.amp_imitation_reward(d)
    ap = RR.AnymalRewardParams()
    ro = dict(lin=rng.normal(size=(N, 3)), ang=rng.normal(size=(N, 3)), cmd=rng.uniform(-1, 1, (N, 3)),
              qvel=rng.normal(size=(N, 12)), qacc=rng.normal(size=(N, 12), scale=10),
              torques=rng.normal(size=(N, 12), scale=20), arate=rng.normal(size=(N, 12)),
              coll=rng.integers(0, 4, N).astype(float), air=rng.uniform(0, 1, (N, 4)))
    ror = RR.anymal_reward(ro["lin"], ro["ang"], ro["cmd"], ro["qvel"], ro["qacc"], ro["torques"],
                           ro["arate"], ro["coll"], ro["air"], ap, variant="rough")
    arrays = {**{f"tri_{k}": v for k, v in tri.items()}, "tri_reward": trr,
              **{f"ing_{k}": v for k, v in ing.items()}, "ing_reward": igr,
              "amp_d": d, "amp_reward": amr,
              **{f"rough_{k}": v for k, v in ro.items()}, "rough_reward": ror}
    save("rewards_extra", {"kind": "rewards", "n": N}, arrays)


if __name__ == "__main__":
    main()
