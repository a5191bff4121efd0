"""Dev tool: a few step-kernel launches for ncu (Ant analog)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2108_10470_b200 import models as M
from paper_2108_10470_b200.scene import Scene
E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
model = sys.argv[3] if len(sys.argv) > 3 else "quadruped"
s = Scene([getattr(M, model)()], E, precision=prec)
s.pos[:, 2] += {"quadruped": 0.37, "quadruped12": 0.34, "humanoid": 1.44}.get(model, 0.5)
s.forward_kinematics()
a = torch.rand(E, s.dofs_per_env, device="cuda") * 2 - 1
for _ in range(4):
    s.step(2, actions=a, action_scale=0.6)
torch.cuda.synchronize()
