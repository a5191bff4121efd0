"""Small-E driver for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library at a few envs.

    compute-sanitizer --tool racecheck python tools/sanitize_drive.py

Covers the fused step kernel (specialised star topologies with the task tail,
the generic kernel with pairs / tendons, the large-articulation variant), the
fp64 path, the indexed setters + FK, refresh, contact geometry / collide, the
task reset, domain randomisation, random forces and the reward kernels.  A
restitution > 0 scene (quadruped_drop's parameters) exercises the freeze-time
restitution target that the plane-overlap path must not race on.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_10470_b200 import models as M  # noqa: E402
from paper_2108_10470_b200.buffers import SimBuffers  # noqa: E402
from paper_2108_10470_b200.envs import make_env  # noqa: E402
from paper_2108_10470_b200.params import SimParams  # noqa: E402
from paper_2108_10470_b200.scene import Scene  # noqa: E402

E = int(os.environ.get("SAN_ENVS", "20"))
only = os.environ.get("SAN_ONLY", "")


def want(name):
    return not only or name in only.split(",")


def env_steps(task, steps=3, **kw):
    env = make_env(task, num_envs=E, seed=0, **kw)
    g = torch.Generator(device="cuda").manual_seed(0)
    for _ in range(steps):
        a = torch.rand((E, env.act_dim), generator=g, device="cuda", dtype=env.scene.dtype) * 2 - 1
        env.step(a)
    env.reset([0, E - 1])
    torch.cuda.synchronize()
    env.close()
    print("ok", task, kw, flush=True)


if want("envs"):
    env_steps("quadruped")                          # Ant analog: star sweep + task tail
    env_steps("quadruped", precision="fp64")
    env_steps("quadruped-anymal-obs")               # 3-joint chains
    env_steps("humanoid")                           # large-articulation variant
if want("dr"):
    env_steps("quadruped", randomize=True, obs_noise=True)
if want("restitution"):
    # restitution > 0: the freeze-time bounce target (plane overlap path)
    p = SimParams(dt=1 / 120, restitution=0.5)
    s = Scene([M.quadruped()], E, p)
    s.pos[:, 2] += 0.5
    s.linvel[:, 2] = -3.0
    for _ in range(4):
        s.step(2)
    torch.cuda.synchronize()
    print("ok restitution", flush=True)
if want("buffers"):
    s = Scene([M.quadruped()], E, SimParams(dt=1 / 120))
    buf = SimBuffers(s)
    root = s.root_state.clone()
    root[:, 2] += 0.1
    buf.set_root_state(root, np.arange(0, E, 3))
    dof = s.dof_state.clone()
    dof[:, 0] = 0.05
    buf.set_dof_state(dof, np.arange(1, E, 2))
    s.forward_kinematics()
    s.refresh_buffers()
    s.contact_geometry()
    s.collide()
    torch.cuda.synchronize()
    print("ok buffers/fk/collide", flush=True)
if want("pairs"):
    import pair_scenes as PS  # authored pair scenes (box / capsule / sphere pairs)
    for name in ("box_stack", "capsule_cross", "franka_cube_stack"):
        s = Scene(PS.SCENES[name][0](), 4, SimParams(dt=1 / 120), shape_pairs="all")
        PS.setup(name, s, jitter=0.3)
        for _ in range(2):
            s.step(1)
        s.collide()
        torch.cuda.synchronize()
        print("ok pairs", name, flush=True)
if want("rewards"):
    from paper_2108_10470_b200 import rewards as R
    n, d = E, torch.device("cuda")
    z = lambda *sh: torch.zeros(*sh, device=d)  # noqa: E731
    R.locomotion_reward(z(n, 3), torch.ones(n, 3, device=d), torch.ones(n, device=d), torch.ones(n, device=d),
                        z(n, 8), z(n, 8), z(n, 8), -torch.ones(8, device=d), torch.ones(8, device=d),
                        torch.ones(n, 8, device=d), z(n), R.LocomotionRewardParams(dt=1 / 60))
    torch.cuda.synchronize()
    print("ok rewards", flush=True)
print("SANITIZE_DRIVE_DONE", flush=True)
