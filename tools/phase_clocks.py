"""DEV TOOL (timing experiment): thread-0 cycles per step_kernel phase,
averaged over CTAs.  Needs the library built with -DBSIM_EXP_PHASE_CLOCKS
(variant `phaseclk`):

    BSIM_NVCC_EXTRA=-DBSIM_EXP_PHASE_CLOCKS python -m paper_2108_10470_b200.build --force
    BSIM_LIB_VARIANT=phaseclk python tools/phase_clocks.py [task] [envs]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_10470_b200 import _native as N  # noqa: E402
from paper_2108_10470_b200.envs import make_env  # noqa: E402

PHASES = ("slab load + sweep-SMSP claim", "stage + actions", "substeps (physics)", "readout + state stores",
          "task tail (reward / done / reset / obs)", "obs copy-out")


def main(task="quadruped", E=16384, steps=20):
    fn = N.lib().bsim_exp_phase_clocks
    fn.argtypes = [C.POINTER(C.c_ulonglong)]
    buf = (C.c_ulonglong * 8)()
    env = make_env(task, num_envs=int(E), seed=0)
    gen = torch.Generator(device="cuda").manual_seed(0)
    for _ in range(5):
        env.step(torch.rand((int(E), env.act_dim), generator=gen, device="cuda") * 2 - 1)
    torch.cuda.synchronize()
    fn(buf)
    for _ in range(steps):
        env.step(torch.rand((int(E), env.act_dim), generator=gen, device="cuda") * 2 - 1)
    torch.cuda.synchronize()
    fn(buf)
    n = max(int(buf[7]), 1)
    print(f"{task} E={E}: {n / steps:.0f} CTAs per launch")
    for i, name in enumerate(PHASES):
        print(f"  {name:40s} {buf[i] / n:9.0f} cycles/CTA  ({buf[i] / n / 1965:.2f} us)")


if __name__ == "__main__":
    main(*sys.argv[1:3])
