"""DEV TOOL: one launch of every non-step kernel at the headline size
(16384 Ant-analog envs, fp32) for an ncu capture:

    ncu --set full -k regex:"task_reset|fk_kernel|set_root|set_dof|refresh|contact_geometry|collide|scan|randomize|force|loco|anymal|cube|franka" \
        python tools/aux_kernels_drive.py

Prints, per kernel family, the algorithmic bytes one launch must move (the
arrays it reads + writes, counted from the shapes) so tools/aux_kernels_md.py
can put achieved GB/s next to the ncu DRAM bytes and duration.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_10470_b200 import rewards as R  # noqa: E402
from paper_2108_10470_b200.envs import make_env  # noqa: E402
from paper_2108_10470_b200.randomize import RandomForceState, random_object_force  # noqa: E402

E = int(os.environ.get("AUX_ENVS", "16384"))
F = 4                                           # fp32 bytes


def main():
    env = make_env("quadruped", num_envs=E, seed=0, randomize=True)
    s = env.scene
    B, D, A = s.bodies_per_env, s.dofs_per_env, s.actors_per_env
    J, P = s.layout.joints_per_env, s.layout.planes_per_env
    algo = {}
    torch.cuda.synchronize()
    # auto-reset of every env: DR (randomize_kernel) + task_reset_kernel (RNG, FK, repack, obs)
    env.reset()
    torch.cuda.synchronize()
    algo["task_reset_kernel"] = E * (B * 13 * F * 2 + D * 2 * F + B * 13 * F + 13 * F + env.obs_dim * F + 64)
    # indexed setters + FK over the touched envs (buffers.py:127-178)
    idx = torch.arange(0, E, 4, device="cuda")
    root = s.root_state.clone()
    root[:, 2] += 0.05
    env.buffers.set_root_state(root, idx)
    dof = s.dof_state.clone()
    env.buffers.set_dof_state(dof, idx)
    torch.cuda.synchronize()
    n = len(idx)
    algo["set_root_kernel"] = n * (13 * F * 2 + 8)
    algo["set_dof_kernel"] = n * (D * 2 * F * 2 + 8)
    algo["fk_kernel"] = n * (B * 13 * F * 2 + D * 2 * F + B * 13 * F + 13 * F)
    s.refresh_buffers()
    algo["refresh_kernel"] = E * (B * 13 * F + B * 13 * F + A * 13 * F + D * 2 * F)
    s.contact_geometry()
    algo["contact_geometry_kernel"] = E * (B * 7 * F + P * (1 + 4 * F + 6 * F + 4 * F))
    s.collide_tensors()
    algo["collide_count_kernel"] = E * B * 7 * F
    torch.cuda.synchronize()
    # random object force (randomize.py:215-221) on body 0 of every env
    fs = RandomForceState(E, rng=0)
    mass = torch.ones(E, device="cuda")
    random_object_force(fs, mass, 1 / 60, body_force=s.ctrl_body_force, body=0, bodies_per_env=B)
    algo["random_force_kernel"] = E * (3 * F * 2 + F + 3 * F + 16)
    # locomotion reward kernel (rewards.py:78-112) standalone
    z = lambda *sh: torch.zeros(*sh, device="cuda")  # noqa: E731
    R.locomotion_reward(z(E, 3), torch.ones(E, 3, device="cuda"), torch.ones(E, device="cuda"),
                        torch.ones(E, device="cuda"), z(E, D), z(E, D), z(E, D), -torch.ones(D, device="cuda"),
                        torch.ones(D, device="cuda"), torch.ones(E, D, device="cuda"), z(E),
                        R.LocomotionRewardParams(dt=1 / 60))
    algo["loco_kernel"] = E * (3 + 3 + 1 + 1 + 4 * D + 1 + 2) * F
    torch.cuda.synchronize()
    print("AUX_ALGO_BYTES " + json.dumps({"envs": E, "bytes_per_launch": algo}), flush=True)


if __name__ == "__main__":
    main()
