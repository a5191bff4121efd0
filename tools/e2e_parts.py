"""Dev: the pieces of the end-to-end host-buffer step (copy times, host-side
Python time of one step, sync latency).   python tools/e2e_parts.py [task] [E]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2108_10470_b200.envs import make_env  # noqa: E402

task = sys.argv[1] if len(sys.argv) > 1 else "quadruped"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
env = make_env(task, num_envs=E, seed=0)
K = 50


def ev_time(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3


d_act = torch.zeros((E, env.act_dim), device="cuda")
h_act = torch.zeros((E, env.act_dim), pin_memory=True)
h_obs = torch.empty(env.obs.shape, pin_memory=True)
print(f"{task} E={E}")
print(f"  H2D actions {h_act.numel()*4/1e6:.2f} MB   {ev_time(lambda: d_act.copy_(h_act, non_blocking=True)):7.1f} us")
print(f"  D2H obs     {h_obs.numel()*4/1e6:.2f} MB   {ev_time(lambda: h_obs.copy_(env.obs, non_blocking=True)):7.1f} us")
big = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
hbig = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
t = ev_time(lambda: hbig.copy_(big, non_blocking=True))
print(f"  D2H 64 MB {64*1.048576/t*1e3:.1f} GB/s;  H2D 64 MB "
      f"{64*1.048576/ev_time(lambda: big.copy_(hbig, non_blocking=True))*1e3:.1f} GB/s")


def host_time(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(K):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    ts.sort()
    return ts[len(ts) // 2] * 1e6


print(f"  host time env.step (no sync)       {host_time(lambda: env.step(d_act)):7.1f} us")
print(f"  host time step_host(sync=False)    {host_time(lambda: env.step_host(h_act, sync=False)):7.1f} us")
print(f"  host time h_act.to(cuda) + step    {host_time(lambda: env.step(h_act.to('cuda', non_blocking=True))):7.1f} us")
s = torch.cuda.current_stream()
print(f"  empty sync round trip              {host_time(lambda: s.synchronize()):7.1f} us")
env.host_zero_copy = True
print(f"  host time step_host zero-copy (sync=False) {host_time(lambda: env.step_host(h_act, sync=False)):7.1f} us")
env.host_zero_copy = False
env.fused = True
print(f"  device fused step (task tail in the step kernel) {ev_time(lambda: env.step(d_act)):7.1f} us")
env.fused = False
print(f"  device two-launch step                           {ev_time(lambda: env.step(d_act)):7.1f} us")
