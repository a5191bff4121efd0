import sys, numpy as np
sys.path[:0] = ["tests", "."]
import scale_parity as SP
from pair_scenes import oracle_trace, oracle_sensitivity
from golden_util import gpu_outputs, load_gpu_state
from paper_2108_10470_b200.scene import Scene
models, p, meta, arr = oracle_trace("shadow_hand_cube")
s = Scene(models, meta["num_envs"], p, precision="fp32", shape_pairs="all", env_origins=arr["param_env_origins"])
sens = oracle_sensitivity(models, p, meta, arr, seeds=(1, 2, 3, 4))
for t in range(meta["steps"]):
    load_gpu_state(s, arr, t); s.step(); got = gpu_outputs(s)
    for k in ("root_state", "body_state", "net_contact"):
        r = arr[f"out_{k}"][t]; r2 = r.reshape(len(r), -1)
        d = np.abs(got[k].reshape(r2.shape) - r2)
        sc = d / (1e-4 + 1e-4 * SP._magnitude(k, r2))
        S = sens[t][k].reshape(r2.shape)
        over = sc > 10
        for i, j in zip(*np.nonzero(over)):
            print(t, k, i, j, f"ref {r2[i,j]:.6g} gpu {got[k].reshape(r2.shape)[i,j]:.6g} d {d[i,j]:.3g} scaled {sc[i,j]:.1f} S {S[i,j]:.3g} ratio {S[i,j]/d[i,j]:.3f}")
