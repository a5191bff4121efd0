"""DEV TOOL: the Shadow Hand scene's fp32 error on the host build of the
kernel (teacher forced vs the float64 oracle trace): elements of root /
body state and contact force beyond 1e-3 + 1e-3 |ref| (vector norms), and
how many of them the reference itself reproduces under fp32-sized input
noise or with its knife-edge joint-limit decisions re-decided.
BSIM_HK_EXTRA=-D... selects arithmetic experiments."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import scale_parity as SP  # noqa: E402
from pair_scenes import oracle_trace  # noqa: E402


def main(name="shadow_hand_cube"):
    from hostkernel.hk import HostKernel
    from paper_2108_10470_b200.layout import SceneLayout
    from pair_scenes import oracle_sensitivity
    models, p, meta, arr = oracle_trace(name)
    sens = oracle_sensitivity(models, p, meta, arr)
    lsens = oracle_sensitivity(models, p, meta, arr, limit_seeds=tuple(range(1, 17)))
    split = np.zeros(4, int)
    E = meta["num_envs"]
    L = SceneLayout(models, True, "all")
    hk = HostKernel(L, E, p, arr["param_env_origins"], fp64=False)
    B = L.bodies_per_env
    be = np.repeat(np.arange(E), B)
    org = arr["param_env_origins"]
    n_over = n_all = 0
    worst = 0.0
    for t in range(meta["steps"]):
        hk.arr["body_q"][...] = np.concatenate([arr["in_pos"][t] - org[be], arr["in_quat"][t], arr["in_linvel"][t],
                                                arr["in_angvel"][t]], 1)
        hk.arr["friction_anchor"][...] = arr["in__friction_anchor"][t] - org[None]
        for k in ("dof_state", "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
                  "ctrl_body_torque", "dof_mode", "nonfinite"):
            hk.arr[k][...] = arr[f"in_{k}"][t]
        hk.step()
        for k in ("root_state", "body_state", "net_contact"):
            split += np.array(SP.excused_split({k: hk.arr[k].astype(float)}, {k: arr[f"out_{k}"][t]}, sens[t], k,
                                               lsens=lsens[t]))
        for k in ("body_state", "net_contact"):
            g = hk.arr[k].astype(float)
            r = arr[f"out_{k}"][t]
            d = np.abs(g - r)
            sc = d / (1e-3 + 1e-3 * SP._magnitude(k, r))
            n_over += int((sc > 1).sum())
            n_all += sc.size
            worst = max(worst, float(sc.max()))
    print(f"{name} fp32 host [{os.environ.get('BSIM_HK_EXTRA', '')}]: {n_over} of {n_all} beyond 1e-3, worst {worst:.1f}x")
    print(f"  root / body / contact beyond 1e-3: ill-conditioned (input noise) {split[0]}, knife-edge limits "
          f"{split[1]}, unexplained {split[3]}")


if __name__ == "__main__":
    main(*sys.argv[1:2])


def rounded_fp64(name="shadow_hand_cube", round_params=True):
    """float64 arithmetic on fp32-ROUNDED state / controls (/ parameters):
    the error fp32 storage alone causes on this model."""
    from hostkernel.hk import HostKernel
    from paper_2108_10470_b200.layout import SceneLayout
    models, p, meta, arr = oracle_trace(name)
    E = meta["num_envs"]
    L = SceneLayout(models, True, "all")
    hk = HostKernel(L, E, p, arr["param_env_origins"], fp64=True)
    r32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    if round_params:
        for k in ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static", "mu_dynamic",
                  "joint_stiffness", "joint_damping", "joint_armature", "joint_friction", "joint_limit_lo",
                  "joint_limit_hi", "plane_off", "plane_rad", "pair_off", "pair_rad"):
            hk.arr[k][...] = r32(hk.arr[k])
    B = L.bodies_per_env
    be = np.repeat(np.arange(E), B)
    org = arr["param_env_origins"]
    n_over = n_all = 0
    worst = 0.0
    for t in range(meta["steps"]):
        hk.arr["body_q"][...] = r32(np.concatenate([arr["in_pos"][t] - org[be], arr["in_quat"][t],
                                                    arr["in_linvel"][t], arr["in_angvel"][t]], 1))
        hk.arr["friction_anchor"][...] = r32(arr["in__friction_anchor"][t] - org[None])
        for k in ("dof_state", "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
                  "ctrl_body_torque"):
            hk.arr[k][...] = r32(arr[f"in_{k}"][t])
        for k in ("dof_mode", "nonfinite"):
            hk.arr[k][...] = arr[f"in_{k}"][t]
        hk.step()
        for k in ("root_state", "body_state", "net_contact"):
            split += np.array(SP.excused_split({k: hk.arr[k].astype(float)}, {k: arr[f"out_{k}"][t]}, sens[t], k,
                                               lsens=lsens[t]))
        for k in ("body_state", "net_contact"):
            g = hk.arr[k].astype(float)
            r = arr[f"out_{k}"][t]
            sc = np.abs(g - r) / (1e-3 + 1e-3 * SP._magnitude(k, r))
            n_over += int((sc > 1).sum())
            n_all += sc.size
            worst = max(worst, float(sc.max()))
    print(f"{name} fp64 host on fp32-rounded inputs (params rounded: {round_params}): {n_over} of {n_all} "
          f"beyond 1e-3, worst {worst:.1f}x")
