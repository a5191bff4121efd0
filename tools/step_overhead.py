"""DEV TOOL: where the fused env step's time goes outside the kernel.  Times
back-to-back control steps (one event pair around N steps, the CPU free to run
ahead) and per-step event pairs with an L2 flush before each step (bench.py's
method), for env.step (fused) and scene.step (physics only), and the host
(Python) time per env.step call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_10470_b200.envs import make_env  # noqa: E402


def main(task="quadruped", E=16384, n=50):
    E = int(E)
    env = make_env(task, num_envs=E, seed=0)
    a = torch.rand((E, env.act_dim), device="cuda") * 2 - 1
    flush = torch.empty(64 << 20, device="cuda")
    fns = {"env.step": lambda: env.step(a),
           "scene.step": lambda: env.scene.step(env.config.decimation, actions=a, action_scale=env.action_scale,
                                                actions_clipped=env.actions)}
    for name, fn in fns.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t_host = (time.perf_counter() - t0) / n * 1e6
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) / n * 1e3
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for i in range(n):
            flush.zero_()
            evs[i][0].record()
            fn()
            evs[i][1].record()
        torch.cuda.synchronize()
        fl = sum(x.elapsed_time(y) for x, y in evs) / n * 1e3
        print(f"{task:22s} {name:11s} host {t_host:6.1f} us/call   back-to-back {b2b:6.1f} us/step   "
              f"flushed per-step events {fl:6.1f} us/step")


if __name__ == "__main__":
    main(*sys.argv[1:3])
