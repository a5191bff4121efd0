"""Dev tool: time the fused step kernel alone (CUDA events, after warm-up)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2108_10470_b200 import models as M
from paper_2108_10470_b200.scene import Scene

def run(model, E, precision, substeps=2, iters=50):
    s = Scene([getattr(M, model)()], E, precision=precision)
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
    print(f"{model:12s} E={E:6d} {precision} substeps={substeps}: {ms*1e3:8.1f} us/control-step  "
          f"{E/ms*1e3:12.4g} control env-steps/s  {E*substeps/ms*1e3:12.4g} sim env-steps/s", flush=True)

for model in ("quadruped", "quadruped12"):
    for E in (4096, 16384, 65536):
        for prec in ("fp32", "fp64"):
            run(model, E, prec)
