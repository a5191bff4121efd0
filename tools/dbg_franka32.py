"""Dev tool: locate the fp32 deviation in the franka_cube_stack teacher-forced trace."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from pair_scenes import oracle_trace
from golden_util import gpu_outputs, load_gpu_state
from paper_2108_10470_b200.scene import Scene
models, p, meta, arr = oracle_trace("franka_cube_stack")
s = Scene(models, meta["num_envs"], p, precision="fp32", shape_pairs="all", env_origins=arr["param_env_origins"])
B = s.bodies_per_env
for t in range(meta["steps"]):
    load_gpu_state(s, arr, t)
    s.step()
    g = gpu_outputs(s)["body_state"]; w = arr["out_body_state"][t]
    d = np.abs(g - w) / (2e-3 + 2e-3 * np.abs(w)); i = np.unravel_index(np.argmax(d), d.shape)
    print(t, round(float(d.max()), 3), "env", i[0] // B, "body", i[0] % B, "comp", i[1], g[i], w[i])
    if d.max() > 1:
        e = i[0] // B
        print("  env bodies z:", w[e*B:(e+1)*B, 2].round(4))
        print("  got lin/ang of that body", g[i[0], 7:13].round(4), "want", w[i[0], 7:13].round(4))
