"""Dev tool: time the fused step kernel alone (CUDA events, after warm-up).

    python tools/quick_step_bench.py [--models quadruped,quadruped12] [--envs 4096,16384] [--prec fp32] [--generic]
"""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2108_10470_b200 import models as M
from paper_2108_10470_b200.scene import Scene


def run(model, E, precision, substeps=2, iters=50, specialize=True, tag=""):
    s = Scene([getattr(M, model)()], E, precision=precision, specialize=specialize)
    s.pos[:, 2] += 0.37
    s.forward_kinematics()
    a = torch.rand(E, s.dofs_per_env, device="cuda") * 2 - 1
    for _ in range(5):
        s.step(substeps, actions=a, action_scale=0.6)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(iters):
        s.step(substeps, actions=a, action_scale=0.6)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / iters
    print(f"{tag}{model:12s} {'spec' if specialize else 'gen '} E={E:6d} {precision}: {ms*1e3:8.1f} us/control-step  "
          f"{E/ms*1e3:12.4g} control env-steps/s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="quadruped,quadruped12")
    ap.add_argument("--envs", default="4096,16384,65536")
    ap.add_argument("--prec", default="fp32,fp64")
    ap.add_argument("--generic", action="store_true")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    for model in a.models.split(","):
        for E in map(int, a.envs.split(",")):
            for prec in a.prec.split(","):
                run(model, E, prec, tag=a.tag)
                if a.generic:
                    run(model, E, prec, specialize=False, tag=a.tag)
