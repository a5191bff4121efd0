"""Dev: end-to-end host-buffer step variants (per-step sync, pinned buffers).
    python tools/host_step_bench.py [task] [E]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2108_10470_b200.envs import make_env  # noqa: E402

task = sys.argv[1] if len(sys.argv) > 1 else "quadruped"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
K = 50


def timed(fn):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


env = make_env(task, num_envs=E, seed=0)
g = torch.Generator(device="cuda").manual_seed(0)
acts = [torch.rand((E, env.act_dim), generator=g, device="cuda") * 2 - 1 for _ in range(4)]
h_act = [a.cpu().pin_memory() for a in acts]
h_obs = torch.empty(env.obs.shape, pin_memory=True)
h_rew = torch.empty(env.reward.shape, pin_memory=True)
h_done = torch.empty(env.done.shape, dtype=torch.bool, pin_memory=True)


def device_step(i):
    env.step(acts[i % 4])


def old_e2e(i):
    o = env.step(h_act[i % 4].to("cuda", non_blocking=True))
    h_obs.copy_(o.obs, non_blocking=True)
    h_rew.copy_(o.reward, non_blocking=True)
    h_done.copy_(o.done, non_blocking=True)
    torch.cuda.current_stream().synchronize()


def host(i):
    env.step_host(h_act[i % 4])


def task_only(i):
    env._call("bsim_task_step", env.scene._s)


print(f"{task} E={E}")
print(f"  device step            {timed(device_step):8.1f} us")
print(f"  task kernel only       {timed(task_only):8.1f} us")
print(f"  e2e per-step copies    {timed(old_e2e):8.1f} us")
for graph in (False, True):
    env.host_graph = graph
    for fused in (False, True):
        env.host_fused = fused
        for n in (0, 1, 4):
            env.host_chunks = n
            print(f"  step_host graph={graph!s:5} fused={fused!s:5} chunks={env.host_chunk_count()} "
                  f"{timed(host):8.1f} us")

env.host_zero_copy = True
print(f"  step_host zero-copy                  {timed(host):8.1f} us")
env.host_zero_copy = False
