"""Dev tool: eager vs CUDA-graph control steps (device-resident actions)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2108_10470_b200.envs import make_env
for task in ("quadruped", "humanoid"):
    for E in (1024, 4096, 16384):
        for graph in (False, True):
            env = make_env(task, num_envs=E, seed=0)
            if graph:
                env.capture_graph()
            a = torch.rand(E, env.act_dim, device="cuda") * 2 - 1
            for _ in range(5):
                env.step(a)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(100):
                env.step(a)
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / 100
            print(f"{task:10s} E={E:6d} graph={graph!s:5s} {ms*1e3:8.1f} us/step {E/ms*1e3/1e6:8.2f} M env-steps/s", flush=True)
            env.close()
