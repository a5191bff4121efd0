"""Dev tool: a few task-tail launches for ncu (Ant analog, 16384 envs)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10470_b200.envs import make_env  # noqa: E402

env = make_env(sys.argv[1] if len(sys.argv) > 1 else "quadruped", num_envs=16384, seed=0)
a = torch.rand((16384, env.act_dim), device="cuda") * 2 - 1
for _ in range(4):
    env.step(a)
for _ in range(3):
    env._call("bsim_task_step", env.scene._s)
torch.cuda.synchronize()
