"""Worker for tests/test_gpu_multirank.py: one rank of a torchrun-style job
(RANK / WORLD_SIZE / MASTER_* from the environment, gloo so ranks may share
one GPU) stepping its shard of a global env batch through the product env
(make_sharded_env -> fused CUDA control steps with auto-resets), then
gathering obs / reward / done / root state on rank 0."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2108_10470_b200.parallel import make_sharded_env, rollout_stats, shard_range  # noqa: E402


def main(task, total, steps, out):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    env = make_sharded_env(task, total, seed=5, episode_length=20, device="cuda:0")
    lo, hi = shard_range(total, world, rank)
    g = np.random.default_rng(17)
    rec = {k: [] for k in ("obs", "reward", "done", "root")}
    for _ in range(steps):
        a = g.uniform(-1.2, 1.2, (total, env.act_dim))[lo:hi]     # the global action matrix, this rank's rows
        o = env.step(torch.as_tensor(a, dtype=env.scene.dtype))
        rec["obs"].append(o.obs.cpu().numpy().copy())
        rec["reward"].append(o.reward.cpu().numpy().copy())
        rec["done"].append(o.done.cpu().numpy().copy())
        rec["root"].append(env.scene.root_state.cpu().numpy().copy())
    mean_r, finished, n = rollout_stats(o.reward, o.done)      # the only collective next to the step
    parts = [None] * world
    dist.all_gather_object(parts, {k: np.stack(v) for k, v in rec.items()})
    if rank == 0:
        cat = {k: np.concatenate([p[k] for p in parts], axis=1) for k in rec}
        np.savez(out, mean_reward=mean_r, finished=finished, n=n, **cat)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
