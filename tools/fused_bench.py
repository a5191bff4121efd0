"""Dev tool: fused (bsim_env_step) vs two-launch control steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2108_10470_b200 import envs as EV
for task in ("quadruped", "quadruped-anymal-obs", "humanoid"):
    for E in (4096, 16384):
        for fused in (False, True):
            EV.EnvBatch.fused = fused
            env = EV.make_env(task, num_envs=E, seed=0)
            a = torch.rand(E, env.act_dim, device="cuda") * 2 - 1
            for _ in range(5):
                env.step(a)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(50):
                env.step(a)
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / 50
            print(f"{task:22s} E={E:6d} fused={fused!s:5s} {ms*1e3:8.1f} us/step {E/ms*1e3/1e6:8.2f} M/s", flush=True)
            env.close()
