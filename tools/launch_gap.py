"""DEV TOOL (timing experiment, variant `phaseclk`): the idle gap between
consecutive step_kernel launches (block 0's entry - the previous launch's
last CTA exit, %globaltimer), back to back, for env.step vs scene.step."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_10470_b200 import _native as N  # noqa: E402
from paper_2108_10470_b200.envs import make_env  # noqa: E402


def main(task="quadruped", E=16384, n=40):
    E = int(E)
    fn = N.lib().bsim_exp_launch_gap
    fn.argtypes = [C.POINTER(C.c_ulonglong)]
    env = make_env(task, num_envs=E, seed=0)
    a = torch.rand((E, env.act_dim), device="cuda") * 2 - 1
    buf = (C.c_ulonglong * 2)()
    for name, f in (("env.step", lambda: env.step(a)),
                    ("scene.step", lambda: env.scene.step(env.config.decimation, actions=a,
                                                          action_scale=env.action_scale,
                                                          actions_clipped=env.actions))):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        fn(buf)
        for _ in range(n):
            f()
        torch.cuda.synchronize()
        fn(buf)
        print(f"{task} {name:10s}: mean gap between launches {buf[0] / max(buf[1], 1) / 1e3:.1f} us "
              f"over {buf[1]} launches")


if __name__ == "__main__":
    main(*sys.argv[1:3])
