"""Dev: cost of the task tail inside the fused control-step launch (env.step)
vs the physics alone (scene.step), warm and with an L2 flush between steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2108_10470_b200.envs import make_env

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
for task in ("quadruped", "quadruped-anymal-obs"):
    env = make_env(task, num_envs=E, seed=0)
    a = torch.rand((E, env.act_dim), device="cuda") * 2 - 1
    flush = torch.empty(64 << 20, device="cuda")
    def phys():
        env.scene.step(env.config.decimation, actions=a, action_scale=env.action_scale, actions_clipped=env.actions)
    def full():
        env.step(a)
    for name, fn in (("physics", phys), ("env.step fused", full)):
        for fl in (False, True):
            for _ in range(5):
                fn()
            ts = []
            for _ in range(30):
                if fl:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); fn(); e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            print(f"{task:22s} {name:16s} flush={fl!s:5} median {ts[len(ts)//2]:7.1f} us  min {ts[0]:7.1f}")
    print("  resets per step ~", float(env.done.float().mean()) * E)
    env.close()
