"""ctypes binding of the C ABI in include/batchsim_b200.h.

The CUDA library is built in-tree (``paper_2108_10470_b200/_lib/libbsim_b200.so``,
see ``build.py``).  There is no fallback: if the library is missing or a call
fails, a ``NativeError`` is raised.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# BSIM_LIB_VARIANT=ieee loads the IEEE-fp32 build (build.py --ieee: no
# -ftz / approximate divide / sqrt) -- a measurement variant for the fp32
# parity table, same kernels and ABI.
_VARIANT = os.environ.get("BSIM_LIB_VARIANT", "")
LIB_PATH = os.path.join(HERE, "_lib", f"libbsim_b200{'_' + _VARIANT if _VARIANT else ''}.so")


class NativeError(RuntimeError):
    pass


def _joint_fields(real):
    return ([(n, C.c_int32) for n in ("kind", "parent", "child", "dof", "actor", "has_limits",
                                      "pad0", "pad1")] +
            [("axis", real * 3), ("origin_pos", real * 3), ("origin_quat", real * 4),
             ("child_pos", real * 3), ("child_quat", real * 4), ("pad", real * 7)])


def _tendon_fields(real):
    return ([(n, C.c_int32) for n in ("kind", "first", "count", "has_limits", "reaction_body",
                                      "actor", "path_offset", "pad")] +
            [(n, real) for n in ("rest_length", "stiffness", "damping", "limit_lo", "limit_hi",
                                 "limit_stiffness")] + [("pad2", real * 2)])


def _telem_fields(real):
    return [("index", C.c_int32), ("parent", C.c_int32), ("joint", C.c_int32),
            ("pad", C.c_int32), ("v", real * 4)]


def _params_fields(real):
    return [("dt", real), ("position_iterations", C.c_int32), ("velocity_iterations", C.c_int32)] + [
        (n, real) for n in ("max_bias", "restitution", "bounce_threshold", "rest_offset",
                            "friction_offset_threshold", "solver_offset_slop", "max_force",
                            "linear_damping", "angular_damping", "max_linear_velocity",
                            "max_angular_velocity")]


class Joint(C.Structure):
    _fields_ = _joint_fields(C.c_float)


class Joint64(C.Structure):
    _fields_ = _joint_fields(C.c_double)


class Tendon(C.Structure):
    _fields_ = _tendon_fields(C.c_float)


class Tendon64(C.Structure):
    _fields_ = _tendon_fields(C.c_double)


class TendonElem(C.Structure):
    _fields_ = _telem_fields(C.c_float)


class TendonElem64(C.Structure):
    _fields_ = _telem_fields(C.c_double)


class Params(C.Structure):
    _fields_ = _params_fields(C.c_float)


class Params64(C.Structure):
    _fields_ = _params_fields(C.c_double)


LAYOUT_INTS = ("num_envs", "actors_per_env", "bodies_per_env", "dofs_per_env", "joints_per_env",
               "planes_per_env", "pairs_per_env", "sensors_per_env", "tendons_per_env", "env_offset",
               "topology_id", "sched_stages", "sched_width", "sched_flags")
LAYOUT_PTRS = ("joints", "plane_body", "pair_body", "sensor_body", "actor_body_offset",
               "actor_dof_offset", "tendons", "tendon_elems", "spatial_paths", "pair_kind", "pair_ext",
               "sweep_sched")


class Layout(C.Structure):
    _fields_ = [(n, C.c_int32) for n in LAYOUT_INTS] + [(n, C.c_void_p) for n in LAYOUT_PTRS]


STATE_PTRS = ("body_q", "friction_anchor", "nonfinite", "env_origins", "inv_mass", "inertia_local",
              "inv_inertia_local", "gravity", "mu_static", "mu_dynamic", "joint_stiffness",
              "joint_damping", "joint_armature", "joint_friction", "joint_limit_lo", "joint_limit_hi",
              "plane_off", "plane_rad", "pair_off", "pair_rad", "ctrl_dof_force",
              "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force", "ctrl_body_torque",
              "dof_mode", "root_state", "body_state", "dof_state", "net_contact", "dof_force",
              "sensor_forces")


class State(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in STATE_PTRS]


class Actions(C.Structure):
    _fields_ = [("actions", C.c_void_p), ("actions_clipped", C.c_void_p), ("scale", C.c_double),
                ("mode", C.c_int32), ("pad", C.c_int32)]


class HostIO(C.Structure):
    """bsim_host_io_t."""
    _fields_ = [("actions", C.c_void_p), ("obs", C.c_void_p), ("reward", C.c_void_p), ("done", C.c_void_p),
                ("timeout", C.c_void_p), ("poisoned", C.c_void_p), ("n_chunks", C.c_int32), ("fused", C.c_int32)]


_lib = None


def _declare(lib):
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "bsim_abi_version": ([], C.c_int),
        "bsim_last_error": ([], C.c_char_p),
        "bsim_step_smem_per_env": ([P(Layout), C.c_int32, P(C.c_int32), P(C.c_int32)], C.c_int),
        "bsim_step_envs_per_wave": ([P(Layout), C.c_int32, P(C.c_int32)], C.c_int),
        "bsim_host_last_error": ([], C.c_char_p),
        "bsim_host_graph_launch": ([vp, vp, C.c_int64, vp], C.c_int),
        "bsim_host_graph_destroy": ([vp], None),
    }
    for suffix, prm in (("", Params), ("_f64", Params64)):
        sig.update({
            "bsim_step" + suffix: ([P(Layout), P(prm), vp, C.c_int32, P(Actions), vp], C.c_int),
            "bsim_env_step" + suffix: ([P(Layout), P(prm), vp, C.c_int32, P(Actions), vp, vp], C.c_int),
            "bsim_env_step_host" + suffix: ([P(Layout), P(prm), vp, C.c_int32, P(Actions), vp, P(HostIO), vp],
                                            C.c_int),
            "bsim_env_step_host_graph" + suffix: ([P(Layout), P(prm), vp, C.c_int32, P(Actions), vp, P(HostIO),
                                                   vp, P(vp)], C.c_int),
            "bsim_step_range" + suffix: ([P(Layout), P(prm), vp, C.c_int32, P(Actions), C.c_int32, C.c_int32, vp],
                                         C.c_int),
            "bsim_env_step_range" + suffix: ([P(Layout), P(prm), vp, C.c_int32, P(Actions), vp,
                                              C.c_int32, C.c_int32, vp], C.c_int),
            "bsim_forward_kinematics" + suffix: ([P(Layout), vp, vp, C.c_uint32, vp], C.c_int),
            "bsim_refresh_buffers" + suffix: ([P(Layout), vp, vp], C.c_int),
            "bsim_set_root_state_indexed" + suffix: ([P(Layout), vp, vp, vp, C.c_int32, vp, vp, vp], C.c_int),
            "bsim_set_dof_state_indexed" + suffix: ([P(Layout), vp, vp, vp, C.c_int32, vp, vp, vp], C.c_int),
            "bsim_contact_geometry" + suffix: ([P(Layout), P(prm), vp, vp, vp, vp, vp, vp], C.c_int),
            "bsim_collide" + suffix: ([P(Layout), P(prm), vp, C.c_int32] + [vp] * 8, C.c_int),
        })
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """Load the in-tree CUDA library (raises NativeError if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"CUDA extension not built: {LIB_PATH} is missing (run __graft_entry__.build())")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
        from . import _tasks_native  # noqa: F401  (declares the task / reward entry points)
        _tasks_native.declare(_lib)
        if _lib.bsim_abi_version() != 2:
            raise NativeError("ABI version mismatch")
    return _lib


def check(rc, what):
    if rc != 0:
        msg = lib().bsim_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def on_scene_device(fn):
    """Run a method with the owning scene's CUDA device current: the native
    entry points launch on the calling thread's current device (cudaGetDevice),
    so a scene on a non-current GPU must switch to it first (and back)."""
    import functools

    import torch

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        scene = getattr(self, "scene", self)
        idx = scene.device.index
        prev = torch.cuda.current_device()
        if idx is None or idx == prev:
            return fn(self, *args, **kwargs)
        torch.cuda.set_device(idx)
        try:
            return fn(self, *args, **kwargs)
        finally:
            torch.cuda.set_device(prev)
    return wrapper
