"""Loading the reference-generated golden fixtures (tests/golden/*.npz)."""

import glob
import json
import os

import numpy as np

from paper_2108_10470_b200 import models as M
from paper_2108_10470_b200.model import load_model
from paper_2108_10470_b200.params import SimParams

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

STATE = ("pos", "quat", "linvel", "angvel", "_friction_anchor", "nonfinite", "dof_state",
         "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
         "ctrl_body_torque", "dof_mode")
PARAMS = ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static",
          "mu_dynamic", "joint_stiffness", "joint_damping", "joint_armature", "joint_friction",
          "joint_limit_lo", "joint_limit_hi", "plane_off", "plane_rad", "pair_off", "pair_rad")
OUTPUTS = ("root_state", "body_state", "dof_state", "net_contact", "dof_force",
           "sensor_forces", "nonfinite", "pos", "quat", "linvel", "angvel", "_friction_anchor")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(str(z["meta"]))
    return meta, {k: z[k] for k in z.files if k != "meta"}


def physics_cases():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        name = os.path.basename(p)[:-4]
        if "meta" not in np.load(p).files:      # e.g. ppo.npz (tests/test_ppo.py)
            continue
        meta, _ = load(name)
        if meta["kind"] == "physics":
            out.append(name)
    return out


def build_models(meta):
    return [M.get_model(m) if isinstance(m, str) else load_model(m) for m in meta["models"]]


def sim_params(meta):
    d = dict(meta["params"])
    d["gravity"] = tuple(d["gravity"])
    return SimParams(**d)


def load_state(scene, arrays, t, names=STATE, prefix="in_"):
    """Copy recorded arrays at step t into a Scene-like object (numpy attrs)."""
    for k in names:
        dst = getattr(scene, k)
        dst[...] = arrays[f"{prefix}{k}"][t]


def load_params(scene, arrays):
    for k in PARAMS:
        getattr(scene, k)[...] = arrays[f"param_{k}"]


def to_local_f32(arr, t, num_envs, bodies_per_env, prefix="in_"):
    """Fixture state at step t (world frame float64) -> the float32 env-local
    arrays of bsim_state_t (what the CUDA path consumes)."""
    E, B = num_envs, bodies_per_env
    org = arr["param_env_origins"]
    body_env = np.repeat(np.arange(E), B)
    bq = np.zeros((E * B, 13))
    bq[:, 0:3] = arr[f"{prefix}pos"][t] - org[body_env]
    bq[:, 3:7] = arr[f"{prefix}quat"][t]
    bq[:, 7:10] = arr[f"{prefix}linvel"][t]
    bq[:, 10:13] = arr[f"{prefix}angvel"][t]
    out = {"body_q": bq.astype(np.float32),
           "friction_anchor": (arr[f"{prefix}_friction_anchor"][t] - org[None]).astype(np.float32),
           "dof_state": arr[f"{prefix}dof_state"][t].astype(np.float32)}
    if prefix == "in_":
        for k in ("ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
                  "ctrl_body_torque"):
            out[k] = arr[f"in_{k}"][t].astype(np.float32)
        out["dof_mode"] = arr["in_dof_mode"][t].astype(np.int8)
        out["nonfinite"] = arr["in_nonfinite"][t].astype(np.bool_)
    return out


def params_f32(arr):
    out = {}
    for k in PARAMS:
        out[k] = arr[f"param_{k}"].astype(np.float32)
    return out


# Tolerance contract for fp32 CUDA vs the float64 oracle:
# |gpu - ref| <= ATOL + RTOL * |ref| per element, per teacher-forced step.
ATOL = 1e-4
RTOL = 1e-4


def rel_err(got, want, atol=ATOL, rtol=RTOL):
    """max over elements of |got-want| / (atol + rtol*|want|); <= 1 passes."""
    got = np.asarray(got, float)
    want = np.asarray(want, float)
    nan = np.isnan(got) & np.isnan(want)
    d = np.where(nan, 0.0, np.abs(got - want)) / (atol + rtol * np.abs(np.nan_to_num(want)))
    return float(np.max(d)) if d.size else 0.0


def gpu_scene_from_fixture(meta, arr, precision="fp32"):
    """Build a GPU Scene matching a physics fixture and load its parameters."""
    import torch

    from paper_2108_10470_b200.scene import Scene
    s = Scene(build_models(meta), meta["num_envs"], sim_params(meta), spacing=meta["spacing"],
              ground=meta["ground"], env_origins=arr["param_env_origins"], precision=precision)
    for k in PARAMS:
        getattr(s, k).copy_(torch.as_tensor(arr[f"param_{k}"], dtype=s.dtype))
    return s


def load_gpu_state(s, arr, t, prefix="in_"):
    """Fixture state at step t -> the GPU scene (world -> env-local in float64
    first, then rounded to the scene precision)."""
    import torch
    E, B = s.num_envs, s.bodies_per_env
    org = arr["param_env_origins"]
    body_env = np.repeat(np.arange(E), B)
    bq = np.concatenate([arr[f"{prefix}pos"][t] - org[body_env], arr[f"{prefix}quat"][t],
                         arr[f"{prefix}linvel"][t], arr[f"{prefix}angvel"][t]], axis=1)
    s.body_q.copy_(torch.as_tensor(bq, dtype=s.dtype))
    s._friction_anchor.copy_(torch.as_tensor(arr[f"{prefix}_friction_anchor"][t] - org[None], dtype=s.dtype))
    s.dof_state.copy_(torch.as_tensor(arr[f"{prefix}dof_state"][t], dtype=s.dtype))
    if prefix == "in_":
        for k in ("ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
                  "ctrl_body_torque"):
            getattr(s, k).copy_(torch.as_tensor(arr[f"in_{k}"][t], dtype=s.dtype))
        s.dof_mode.copy_(torch.as_tensor(arr["in_dof_mode"][t].astype(np.int8)))
        s.nonfinite.copy_(torch.as_tensor(arr["in_nonfinite"][t]))


def gpu_outputs(s):
    """Scene outputs as float64 numpy in the reference frame (world)."""
    out = {k: getattr(s, k).double().cpu().numpy() for k in
           ("root_state", "body_state", "dof_state", "net_contact", "dof_force", "sensor_forces")}
    out["nonfinite"] = s.nonfinite.cpu().numpy()
    out["_friction_anchor"] = s._friction_anchor.double().cpu().numpy() + s.env_origins_host[None]
    return out
