"""DEV TOOL: the Shadow Hand / Franka env step (fused task tail, resets with
DR) vs the physics launch alone, back to back, and the reset count per step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_10470_b200.envs import make_env  # noqa: E402


def main(E=16384, n=20):
    for name, kw, EE in (("shadow-hand", {"randomize": True}, int(E)), ("shadow-hand", {}, int(E)),
                         ("franka-cube-stack", {}, int(E) // 2)):
        env = make_env(name, num_envs=EE, seed=0, **kw)
        s = env.scene
        g = torch.Generator(device="cuda").manual_seed(0)
        acts = [torch.rand((EE, env.act_dim), generator=g, device="cuda", dtype=s.dtype) * 2 - 1 for _ in range(4)]
        for i in range(5):
            env.step(acts[i % 4])
        torch.cuda.synchronize()
        resets = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            o = env.step(acts[i % 4])
            resets += o.done
        e1.record()
        torch.cuda.synchronize()
        t_env = e0.elapsed_time(e1) / n * 1e3
        e0.record()
        for i in range(n):
            s.step(env.config.decimation, actions=acts[i % 4], action_scale=env.action_scale,
                   actions_clipped=env.actions)
        e1.record()
        torch.cuda.synchronize()
        t_phys = e0.elapsed_time(e1) / n * 1e3
        print(f"{name} {kw} E={EE}: env.step {t_env:.0f} us, physics only {t_phys:.0f} us, "
              f"resets per step {int(resets.sum()) / n:.1f}")


if __name__ == "__main__":
    main(*sys.argv[1:2])
