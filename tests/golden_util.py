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
