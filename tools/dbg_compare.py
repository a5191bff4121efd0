"""Dev tool: GPU step vs host build of the same kernel body on a fixture."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from golden_util import *
from hostkernel.hk import HostKernel
from paper_2108_10470_b200.layout import SceneLayout
case = sys.argv[1]; prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
meta, arr = load(case)
s = gpu_scene_from_fixture(meta, arr, prec)
load_gpu_state(s, arr, 0)
L = SceneLayout(build_models(meta), meta["ground"]); E = meta["num_envs"]
hk = HostKernel(L, E, sim_params(meta), arr["param_env_origins"], fp64=(prec == "fp64"))
for k in PARAMS: hk.arr[k][...] = arr[f"param_{k}"]
for name in ("body_q", "dof_state", "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target",
             "ctrl_body_force", "ctrl_body_torque", "dof_mode", "nonfinite"):
    hk.arr[name][...] = getattr(s, name).cpu().numpy()
hk.arr["friction_anchor"][...] = s._friction_anchor.cpu().numpy()
s.step(); hk.step()
for k in ("body_q", "dof_state", "net_contact", "dof_force", "root_state"):
    g = getattr(s, k).double().cpu().numpy(); h = hk.arr[k]
    d = np.abs(g - h)
    print(k, "maxdiff", np.nanmax(d) if d.size else 0)
    if d.size and np.nanmax(d) > 1e-6:
        i = np.unravel_index(np.nanargmax(d), d.shape); print("  at", i, g[i], h[i])
        print("  gpu row", np.round(g[i[0]], 5)); print("  host row", np.round(h[i[0]], 5))
