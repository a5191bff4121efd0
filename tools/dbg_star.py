"""Dev: star (AOT two-lane) sweep vs the generic sweep, one step, per-body diffs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2108_10470_b200 import models as M
from paper_2108_10470_b200.scene import Scene
a = Scene([M.quadruped()], 64, precision="fp64")
b = Scene([M.quadruped()], 64, precision="fp64", specialize=False)
g = np.random.default_rng(5)
for s in (a, b):
    s.pos[:, 2] += float(os.environ.get("DZ", "0.37"))
    s.forward_kinematics()
for it in range(int(os.environ.get("NSTEP", "6"))):
    act = torch.as_tensor(g.uniform(-1, 1, (64, a.dofs_per_env)), device="cuda")
    for sub in (1, 2):
        pass
    a.step(1, actions=act, action_scale=0.6)
    b.step(1, actions=act, action_scale=0.6)
    da = (a.body_q - b.body_q).abs().view(64, 9, 13).amax(0).cpu().numpy()
    print("step", it, "max per body [pos quat v w]:")
    for body in range(9):
        print("  body", body, np.array2string(np.array([da[body, 0:3].max(), da[body, 3:7].max(), da[body, 7:10].max(),
                                                      da[body, 10:13].max()]), precision=2))
    nc = (a.net_contact - b.net_contact).abs().max().item()
    print("  net_contact", nc)
    if da.max() > 1e-9:
        break
