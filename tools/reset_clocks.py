"""DEV TOOL (timing experiment): cycles per phase of the fused auto-reset.
Needs the library built with -DBSIM_EXP_RESET_CLOCKS (variant `resetclk`):

    BSIM_NVCC_EXTRA=-DBSIM_EXP_RESET_CLOCKS python -m paper_2108_10470_b200.build --force
    BSIM_LIB_VARIANT=resetclk python tools/reset_clocks.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_10470_b200 import _native as N  # noqa: E402
from paper_2108_10470_b200.envs import make_env  # noqa: E402

PHASES = ("clear + DR", "RNG + root/DOF draws", "obs noise", "FK", "repack", "post-reset")


def main(task="quadruped", E=16384, steps=30):
    lib = N.lib()
    fn = lib.bsim_exp_reset_clocks
    fn.argtypes = [C.POINTER(C.c_ulonglong)]
    env = make_env(task, num_envs=E, seed=0)
    gen = torch.Generator(device="cuda").manual_seed(0)
    buf = (C.c_ulonglong * 8)()
    for _ in range(5):
        env.step(torch.rand((E, env.act_dim), generator=gen, device="cuda") * 2 - 1)
    torch.cuda.synchronize()
    fn(buf)
    knock = torch.arange(0, E, 50, device="cuda")      # 2 % of the envs fall every step: resets at the next
    for _ in range(steps):
        root = env.scene.root_state.clone()
        root[:, 2] = 0.05
        env.buffers.set_root_state(root, knock)
        env.step(torch.rand((E, env.act_dim), generator=gen, device="cuda") * 2 - 1)
    torch.cuda.synchronize()
    fn(buf)
    n = max(int(buf[7]), 1)
    print(f"{task} E={E}: {n} resets in {steps} steps ({n / steps:.1f} per step)")
    tot = 0
    for i, name in enumerate(PHASES):
        cyc = buf[i] / n
        tot += cyc
        print(f"  {name:22s} {cyc:10.0f} cycles/reset  ({cyc / 1965:.2f} us at 1965 MHz)")
    print(f"  {'total':22s} {tot:10.0f} cycles/reset  ({tot / 1965:.2f} us)")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []))
