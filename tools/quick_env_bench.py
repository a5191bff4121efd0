"""Dev tool: time EnvBatch.step (the fused control step) per task with CUDA
events after warm-up:  python tools/quick_env_bench.py humanoid:16384 franka-cube-stack:8192 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_10470_b200.envs import make_env  # noqa: E402


def run(task, E, iters=30):
    env = make_env(task, num_envs=E, seed=0)
    gen = torch.Generator(device=env.obs.device).manual_seed(1)
    acts = [torch.rand((E, env.act_dim), generator=gen, device=env.obs.device, dtype=env.scene.dtype) * 2 - 1
            for _ in range(4)]
    for i in range(5):
        env.step(acts[i % 4])
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for i in range(iters):
        env.step(acts[i % 4])
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / iters
    print(f"{os.environ.get('BSIM_LIB_VARIANT', '-'):6s} {task:20s} E={E:6d}: {ms * 1e3:8.1f} us/control-step "
          f"{E / ms * 1e3 / 1e6:7.2f} M env-steps/s", flush=True)
    env.close()


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        task, E = spec.split(":")
        run(task, int(E))
