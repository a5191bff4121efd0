"""Authored scenes for the box / capsule pair types (shape_pairs="all"), which
the reference does not have (parity unpinned).  Traces are
produced by the float64 C oracle (oracle/bso.c, an independent restatement of
the same narrow phase) in the golden-fixture format of tests/golden_util.py,
so the host build of the kernel body and the CUDA path are compared against
it exactly like the reference-generated fixtures."""

import numpy as np

from paper_2108_10470_b200 import models as M
from paper_2108_10470_b200.model import load_model
from paper_2108_10470_b200.models import capsule_inertia
from paper_2108_10470_b200.params import SimParams

G = 9.81


def capsule(name, m, r, hh, fixed=False):
    return load_model({"name": name, "fixed_base": fixed,
                       "links": [{"name": "c", "mass": m, "inertia": list(capsule_inertia(m, r, hh)),
                                  "shape": {"kind": "capsule", "params": [r, hh]}}]})


def q_axis(ax, ang):
    ax = np.asarray(ax, float)
    ax = ax / np.linalg.norm(ax)
    return np.r_[ax * np.sin(ang / 2), np.cos(ang / 2)]


SCENES = {
    # box B (rotated) resting on box A resting on the ground: 16 PB corner slots
    "box_stack": (lambda: [M.free_box((0.2, 0.2, 0.1), 2.0), M.free_box((0.1, 0.1, 0.1), 1.0)],
                  [((0, 0, 0.1), (0, 0, 1), 0.0), ((0.05, 0.02, 0.3), (0, 0, 1), 0.3)]),
    # three boxes stacked: 24 plane + 48 PB slots (72 > 64: the sequential
    # sweep's activity mask runs in two 64-slot chunks)
    "box_tower": (lambda: [M.free_box((0.2, 0.2, 0.1), 2.0), M.free_box((0.15, 0.15, 0.1), 1.5),
                           M.free_box((0.1, 0.1, 0.1), 1.0)],
                  [((0, 0, 0.1), (0, 0, 1), 0.0), ((0.02, 0.01, 0.3), (0, 0, 1), 0.1),
                   ((-0.01, 0.02, 0.5), (0, 0, 1), 0.2)]),
    # sphere on a box: 1 PB slot
    "sphere_on_box": (lambda: [M.free_box((0.2, 0.2, 0.1), 2.0), M.free_sphere(0.1, 1.0)],
                      [((0, 0, 0.1), (0, 0, 1), 0.0), ((0.05, 0.0, 0.3), (0, 0, 1), 0.0)]),
    # two horizontal capsules crossing: 1 CC slot
    "capsule_cross": (lambda: [capsule("a", 1.0, 0.05, 0.2), capsule("b", 0.5, 0.05, 0.2)],
                      [((0, 0, 0.05), (0, 1, 0), np.pi / 2), ((0, 0, 0.15), (1, 0, 0), np.pi / 2)]),
    # horizontal capsule on a box: 2 PB (capsule ends) + 8 PC (box corners)
    "capsule_on_box": (lambda: [M.free_box((0.2, 0.2, 0.1), 2.0), capsule("b", 0.5, 0.05, 0.1)],
                       [((0, 0, 0.1), (0, 0, 1), 0.0), ((0, 0, 0.2505), (1, 0, 0), np.pi / 2)]),
    # Franka cube-stack (BASELINE config 4): arm + gripper pads vs two cubes
    # (4 PB pad-cube slots, 16 PB cube-cube slots), cubes on the ground
    "franka_cube_stack": (lambda: [M.franka(), M.cube("cubeA", M.CUBE_A_HALF, 0.3),
                                   M.cube("cubeB", M.CUBE_B_HALF, 0.5)],
                          [((0, 0, 0), (0, 0, 1), 0.0), ((0.45, 0.0, 0.025), (0, 0, 1), 0.3),
                           ((0.45, 0.15, 0.035), (0, 0, 1), -0.2)]),
    # Shadow Hand (BASELINE config 5): 24-DOF hand with coupling tendons, a
    # cube on the palm (16 PB palm-cube + 5 PB fingertip-cube slots)
    "shadow_hand_cube": (lambda: [M.shadow_hand(), M.cube("cube", M.SHADOW_CUBE_HALF, 0.1)],
                         [(M.SHADOW_HAND_ROOT, (0, 0, 1), 0.0),
                          ((0.145, 0.0, M.SHADOW_HAND_ROOT[2] + 0.012 + M.SHADOW_CUBE_HALF + 0.001), (0, 0, 1), 0.2)]),
    # sphere cradled between two static horizontal capsule rails: 2 PC slots
    "sphere_in_cradle": (lambda: [capsule("rail_a", 1.0, 0.05, 0.25, fixed=True),
                                  capsule("rail_b", 1.0, 0.05, 0.25, fixed=True), M.free_sphere(0.08, 0.4)],
                         [((0, -0.06, 0.2), (0, 1, 0), np.pi / 2), ((0, 0.06, 0.2), (0, 1, 0), np.pi / 2),
                          ((0.02, 0.0, 0.3153), (0, 0, 1), 0.0)]),
}


def setup(name, s, jitter=0.0, seed=0):
    """Place the actors of scene `name` (env-local poses + the env origins);
    `jitter` adds per-env random velocities."""
    _, poses = SCENES[name]
    B, E = s.bodies_per_env, s.num_envs
    rng = np.random.default_rng(seed)
    gpu = hasattr(s, "env_origins_host")       # the CUDA Scene keeps env-local positions
    org = np.zeros((E, 3)) if gpu else s.env_origins
    put = (lambda v: __import__("torch").as_tensor(v, dtype=s.dtype)) if gpu else (lambda v: v)  # noqa: E731
    roots = [s.actor_body_offset[a] for a in range(len(poses))] if hasattr(s, "actor_body_offset") \
        else list(s.layout.actor_body_offset)
    for e in range(E):
        for a, (p, ax, ang) in enumerate(poses):
            r = e * B + roots[a]
            s.pos[r] = put(org[e] + np.asarray(p, float))
            s.quat[r] = put(q_axis(ax, ang))
            if jitter and name not in ("franka_cube_stack", "shadow_hand_cube"):
                s.linvel[r] = put(rng.uniform(-jitter, jitter, 3))
                s.angvel[r] = put(rng.uniform(-jitter, jitter, 3))
    if name == "franka_cube_stack":            # arm at its home pose, PD-held
        home = np.tile(M.FRANKA_HOME, E)
        s.dof_state[:, 0] = put(home)
        s.ctrl_dof_pos_target[:] = put(home)
    if s.dofs_per_env:
        s.forward_kinematics()


STATE = ("pos", "quat", "linvel", "angvel", "_friction_anchor", "nonfinite", "dof_state",
         "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
         "ctrl_body_torque", "dof_mode")
OUTPUTS = ("root_state", "body_state", "dof_state", "net_contact", "dof_force", "sensor_forces", "nonfinite",
           "pos", "quat", "linvel", "angvel", "_friction_anchor")


def oracle_trace(name, E=4, steps=12, warm=30, dt=1 / 120, jitter=0.3):
    """(meta, arrays) in the golden-fixture format: the oracle's state before
    / after each of `steps` steps, after `warm` steps of settling."""
    from oracle.oracle import OracleScene
    models = SCENES[name][0]()
    p = SimParams(dt=dt)
    s = OracleScene(models, E, p, shape_pairs="all")
    setup(name, s, jitter=jitter)
    rng = np.random.default_rng(11)
    for _ in range(warm):
        s.step()
    if s.dofs_per_env:                        # random PD targets around the start pose from here on
        s.ctrl_dof_pos_target[:] = s.ctrl_dof_pos_target + 0.3 * rng.uniform(-1, 1, s.num_dofs)
    arr = {f"param_{k}": np.array(getattr(s, k)) for k in
           ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static", "mu_dynamic",
            "joint_stiffness", "joint_damping", "joint_armature", "joint_friction", "joint_limit_lo",
            "joint_limit_hi", "plane_off", "plane_rad", "pair_off", "pair_rad", "env_origins")}
    rec = {f"in_{k}": [] for k in STATE}
    rec.update({f"out_{k}": [] for k in OUTPUTS})
    for _ in range(steps):
        for k in STATE:
            rec[f"in_{k}"].append(np.array(getattr(s, k), copy=True))
        s.step()
        for k in OUTPUTS:
            rec[f"out_{k}"].append(np.array(getattr(s, k), copy=True))
    arr.update({k: np.stack(v) for k, v in rec.items()})
    meta = {"kind": "physics", "num_envs": E, "steps": steps, "params": {"dt": dt}, "spacing": 4.0, "ground": True}
    return models, p, meta, arr


def oracle_sensitivity(models, p, meta, arr, seeds=(1, 2), limit_seeds=()):
    """Per step and output, the element-wise max |oracle(perturbed pre-state) -
    oracle(exact pre-state)| over the fp32 rounding of the pre-state (env-local
    positions, as the CUDA path stores them) and len(seeds) random 2^-24
    relative jitters of it: how far the float64 reference algorithm itself
    moves each output under fp32-sized input noise (tests/scale_parity.py
    `sensitivity`, for these small authored scenes).  With `limit_seeds`
    instead: the exact pre-state with the joint-limit activations the
    reference decides within 8 fp32 ulps of the joint angle re-decided at
    random (scale_parity.limit_sensitivity)."""
    from oracle.oracle import OracleScene
    from scale_parity import LIMIT_MARGIN
    E = meta["num_envs"]
    s = OracleScene(models, E, p, shape_pairs="all", env_origins=arr["param_env_origins"])
    for k in ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static", "mu_dynamic",
              "joint_stiffness", "joint_damping", "joint_armature", "joint_friction", "joint_limit_lo",
              "joint_limit_hi", "plane_off", "plane_rad", "pair_off", "pair_rad"):
        getattr(s, k)[...] = arr[f"param_{k}"]
    org = np.repeat(arr["param_env_origins"], s.bodies_per_env, axis=0)

    def r32(x):
        return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)

    def jitter(seed):
        rng = np.random.default_rng(seed)
        return lambda x: np.asarray(x, np.float64) * (1.0 + rng.uniform(-1, 1, np.shape(x)) * 2.0 ** -24)

    def ident(x):
        return np.asarray(x, np.float64)

    runs = ([(ident, sd) for sd in limit_seeds] if limit_seeds else
            [(r32, None)] + [(jitter(sd), None) for sd in seeds])
    outs = ("root_state", "body_state", "net_contact", "dof_state")
    sens = []
    for t in range(meta["steps"]):
        dev = {k: 0.0 for k in outs}
        for tf, lsd in runs:
            s.limit_jitter = None if lsd is None else (lsd * 1000 + t + 1, LIMIT_MARGIN)
            s.pos[...] = org + tf(arr["in_pos"][t] - org)
            for k in ("quat", "linvel", "angvel", "dof_state"):
                getattr(s, k)[...] = tf(arr[f"in_{k}"][t])
            a = arr["in__friction_anchor"][t]
            s._friction_anchor[...] = arr["param_env_origins"][None] + tf(a - arr["param_env_origins"][None])
            for k in ("ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
                      "ctrl_body_torque", "dof_mode", "nonfinite"):
                getattr(s, k)[...] = arr[f"in_{k}"][t]
            s.step()
            for k in outs:
                dev[k] = np.maximum(dev[k], np.abs(np.asarray(getattr(s, k), float) - arr[f"out_{k}"][t]))
        sens.append(dev)
    return sens
