"""DEV TOOL (timing experiment): per-CTA timeline of ONE step_kernel launch
(variant `phaseclk`: -DBSIM_EXP_PHASE_CLOCKS), physics-only (Scene.step) vs
the fused env step (EnvBatch.step): kernel span, CTA duration spread, the
last CTA's start / tail, per-SM busy time.

    BSIM_LIB_VARIANT=phaseclk python tools/cta_timeline.py [task] [envs]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_10470_b200 import _native as N  # noqa: E402
from paper_2108_10470_b200.envs import make_env  # noqa: E402


def grab(fn, n):
    buf = (C.c_ulonglong * (4096 * 4))()
    fn(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 4)[:n].astype(np.int64)
    return a


def report(name, a):
    sm, t0, tt, t1 = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    base = t0.min()
    t0, tt, t1 = (t0 - base) / 1e3, (tt - base) / 1e3, (t1 - base) / 1e3
    dur = t1 - t0
    tail = t1 - tt
    span = t1.max()
    busy = np.zeros(sm.max() + 1)
    np.add.at(busy, sm, dur)
    late = np.argsort(t1)[-5:]
    print(f"{name}: {len(a)} CTAs, span {span:.1f} us, CTA duration mean {dur.mean():.1f} p50 {np.median(dur):.1f} "
          f"p99 {np.percentile(dur, 99):.1f} max {dur.max():.1f} us; tail mean {tail.mean():.2f} max {tail.max():.2f} us")
    print(f"   start times: first wave ends by {np.sort(t0)[592] if len(t0) > 592 else 0:.1f} us; last CTA start "
          f"{t0.max():.1f} us; per-SM busy mean {busy[busy > 0].mean():.1f} max {busy.max():.1f} us / 4 slots")
    for i in late:
        print(f"   late CTA {i}: sm {sm[i]} start {t0[i]:.1f} end {t1[i]:.1f} dur {dur[i]:.1f} tail {tail[i]:.2f}")


def main(task="quadruped", E=16384):
    E = int(E)
    fn = N.lib().bsim_exp_cta_times
    fn.argtypes = [C.POINTER(C.c_ulonglong)]
    env = make_env(task, num_envs=E, seed=0)
    gen = torch.Generator(device="cuda").manual_seed(0)
    a = torch.rand((E, env.act_dim), generator=gen, device="cuda") * 2 - 1
    flush = torch.empty(64 << 20, device="cuda")
    for mode in ("physics", "fused", "physics", "fused"):
        for _ in range(3):
            flush.zero_()
            if mode == "physics":
                env.scene.step(env.config.decimation, actions=a, action_scale=env.action_scale,
                               actions_clipped=env.actions)
            else:
                env.step(a)
        torch.cuda.synchronize()
        n = int(os.environ.get("CTAS", "0")) or 4096
        arr = grab(fn, n)
        arr = arr[arr[:, 1] > 0]
        report(f"{task} {mode}", arr[arr[:, 1] >= arr[:, 1].max() - 10_000_000])   # this launch's CTAs


if __name__ == "__main__":
    main(*sys.argv[1:3])
