"""Contact masks and the collide() list at BASELINE.json scale, bit-exact.

North star: "contact-pair counts, indices and reset masks must be bit-exact".
The reference evaluates every candidate slot against the current poses and
keeps `depth > -solver_offset_slop` (physics.py:463-498), and `collide()`
lists the active slots planes first, then pairs, slot-major and
env-ascending (physics.py:500-517).  Here, at 4096 and 16384 envs of the Ant
and ANYmal analogs and of the authored multi-actor scene (sphere-sphere
pairs, capsules, boxes), the float64 oracle is run to a contact-rich state
(drops from random heights, random PD targets), that state is rounded to the
device precision and given to BOTH sides, and:

  * the active mask of every (slot, env) is equal, except inside the band
    |depth + slop| < eps where the device's own rounding of the slot centre
    decides a tie (eps = 1e-6 m fp32, 1e-12 m fp64; ties are counted and
    reported, and must be rare);
  * the compacted list (`bsim_collide`: count, body_a, body_b) equals the
    oracle's active list entry for entry (tie entries removed from both);
  * the device list equals the device mask compacted on the host (its own
    order and count, exactly, ties included).
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SCENES = ("quadruped", "quadruped12", "kitchen_sink")


def _models(name):
    from paper_2108_10470_b200 import models as M
    if name == "kitchen_sink":
        from golden_util import build_models, load, sim_params
        meta, _ = load("kitchen_sink")
        return build_models(meta), sim_params(meta), meta.get("ground", True)
    from paper_2108_10470_b200.params import SimParams
    return [getattr(M, name)()], SimParams(dt=1 / 120), True


def _contact_rich_state(name, E, seed=0, warm=8):
    from oracle.oracle import OracleScene
    models, params, ground = _models(name)
    ref = OracleScene(models, E, params, ground=ground, threads=os.cpu_count() or 1)
    rng = np.random.default_rng(seed)
    A = ref.actors_per_env
    for a in range(A):             # drop every actor root from a random height (some start in the ground)
        rows = np.arange(E) * ref.bodies_per_env + ref.actor_body_offset[a]
        ref.pos[rows, 2] += rng.uniform(-0.15, 0.45, E)
    ref.forward_kinematics()
    for _ in range(warm):
        ref.ctrl_dof_pos_target[:] = rng.uniform(-0.6, 0.6, ref.num_dofs)
        ref.step()
    return ref, models, params, ground


def _round_into(ref, gpu):
    """Round the oracle's state to the device precision (env-local, as the
    device stores it) and write the rounded values back into the oracle."""
    B = ref.bodies_per_env
    be = np.repeat(np.arange(ref.num_envs), B)
    org = ref.env_origins
    dt = np.float32 if gpu.dtype == torch.float32 else np.float64
    local = (ref.pos - org[be]).astype(dt).astype(np.float64)
    quat = ref.quat.astype(dt).astype(np.float64)
    ref.pos[:] = org[be] + local
    ref.quat[:] = quat
    bq = np.concatenate([local, quat, ref.linvel, ref.angvel], 1)
    gpu.body_q.copy_(torch.as_tensor(bq, dtype=gpu.dtype))


def _oracle_list(act, L, E, B):
    """(body_a, body_b) of the active slots in collide() order."""
    ba, bb = [], []
    P = L.planes_per_env
    for i in range(P + L.pairs_per_env):
        for e in np.nonzero(act[i * E:(i + 1) * E])[0]:
            if i < P:
                ba.append(-1)
                bb.append(e * B + L.plane_body[i])
            else:
                pa, pb = L.pair_body[i - P]
                ba.append(e * B + pa)
                bb.append(e * B + pb)
    return np.asarray(ba, np.int64), np.asarray(bb, np.int64)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("E", [4096, 16384])
@pytest.mark.parametrize("name", SCENES)
def test_contact_masks_and_collide_list_bit_exact(name, E, precision):
    from paper_2108_10470_b200.scene import Scene
    ref, models, params, ground = _contact_rich_state(name, E)
    gpu = Scene(models, E, params, ground=ground, precision=precision)
    _round_into(ref, gpu)
    L, B = gpu.layout, gpu.bodies_per_env
    act_o, depth_o, _, _ = ref.contact_geometry()
    act_g, depth_g, _, _ = gpu.contact_geometry()
    act_g = act_g.cpu().numpy()
    eps = 1e-6 if precision == "fp32" else 1e-12
    tie = np.abs(depth_o + params.solver_offset_slop) < eps
    n_active = int(act_o.sum())
    assert n_active > 0.2 * E, "state should be contact rich"
    assert (~act_o).sum() > 0.2 * E, "and have inactive slots"
    mismatch = act_o != act_g
    assert not np.any(mismatch & ~tie), (name, E, int((mismatch & ~tie).sum()))
    assert tie.sum() <= max(4, 1e-4 * tie.size), (name, int(tie.sum()))      # ties are rare
    # the compacted list vs the oracle's, entry for entry
    k, ba, bb, depth, point, normal = gpu.collide_tensors()
    ba, bb = ba.cpu().numpy().astype(np.int64), bb.cpu().numpy().astype(np.int64)
    oa, ob = _oracle_list(act_o, L, E, B)
    ga, gb = _oracle_list(act_g, L, E, B)
    assert k == len(ga) and np.array_equal(ba, ga) and np.array_equal(bb, gb)   # device list == device mask
    if not mismatch.any():
        assert k == n_active and np.array_equal(ba, oa) and np.array_equal(bb, ob)
    else:                                                   # drop the tie slots from both lists
        keep_o = _oracle_list(act_o & ~mismatch, L, E, B)
        keep_g = _oracle_list(act_g & ~mismatch, L, E, B)
        assert all(np.array_equal(x, y) for x, y in zip(keep_o, keep_g))
    print(f"{name} E={E} {precision}: {n_active} active of {act_o.size} slots, {int(tie.sum())} in the tie band, "
          f"{int(mismatch.sum())} decided differently")
