"""DEV TOOL (timing experiment, variant `passclk`: -DBSIM_EXP_PASS_CLOCKS):
thread-0 cycles per solver pass in phase A / the sweep / the tail items,
averaged over CTAs and passes, for the physics launch (Scene.step)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_10470_b200 import _native as N  # noqa: E402
from paper_2108_10470_b200 import models as M  # noqa: E402
from paper_2108_10470_b200.scene import Scene  # noqa: E402


def main(model="quadruped", E=16384):
    E = int(E)
    f0, f1 = N.lib().bsim_exp_pass_clocks, N.lib().bsim_exp_pass_clocks_large
    for f in (f0, f1):
        f.argtypes = [C.POINTER(C.c_ulonglong)]
    buf = (C.c_ulonglong * 8)()

    def fn(out):              # both TUs' counters (the default and the large-articulation kernels)
        tmp = (C.c_ulonglong * 8)()
        f0(out)
        f1(tmp)
        for i in range(8):
            out[i] += tmp[i]
    if model in ("shadow-hand", "franka-cube-stack"):
        from paper_2108_10470_b200.envs import make_env
        s = make_env(model, num_envs=E, seed=0).scene
    else:
        s = Scene([getattr(M, model)()], E)
        s.pos[:, 2] += {"quadruped": 0.37, "quadruped12": 0.34, "humanoid": 1.44}.get(model, 0.5)
        s.forward_kinematics()
    a = torch.rand(E, s.dofs_per_env, device="cuda") * 2 - 1
    for _ in range(5):
        s.step(2, actions=a, action_scale=0.6)
    torch.cuda.synchronize()
    fn(buf)
    for _ in range(10):
        s.step(2, actions=a, action_scale=0.6)
    torch.cuda.synchronize()
    fn(buf)
    n = max(int(buf[7]), 1)
    names = ("phase A (items + barrier)", "star sweep (+ overlap work, barrier)",
             "star tail items / generic sweep (+ barrier)")
    print(f"{model} E={E}: {n} CTA-passes")
    for i, nm in enumerate(names):
        print(f"  {nm:40s} {buf[i] / n:8.0f} cycles per pass")


if __name__ == "__main__":
    main(*sys.argv[1:3])
