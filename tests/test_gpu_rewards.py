"""Device reward kernels vs the reference's batched rewards (golden `rewards`,
random inputs incl. limit-adjacent DOFs, near-success quaternions and
stacked cubes)."""

import numpy as np
import pytest

from golden_util import load, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_reward_kernels_match_reference(dtype):
    from paper_2108_10470_b200 import rewards as R
    _, a = load("rewards")
    tol = 1e-10 if dtype == np.float64 else 2e-5
    c = lambda k: a[k].astype(dtype)  # noqa: E731
    r, pot = R.locomotion_reward(c("loc_torso"), c("loc_target"), c("loc_up"), c("loc_heading"), c("loc_actions"),
                                 c("loc_dof_pos"), c("loc_dof_vel"), c("loc_lo"), c("loc_hi"), c("loc_strength"),
                                 c("loc_prev"), R.LocomotionRewardParams(dt=1 / 60))
    assert rel_err(r.double().cpu().numpy(), a["loc_reward"], tol, tol) <= 1
    assert rel_err(pot.double().cpu().numpy(), a["loc_potential"], tol, tol) <= 1
    ar = R.anymal_reward(c("any_lin"), c("any_ang"), c("any_cmd"), None, None, c("any_torques"), None, None, None,
                         R.AnymalRewardParams(dt=1 / 60))
    assert rel_err(ar.double().cpu().numpy(), a["any_reward"], tol, tol) <= 1
    cr, _, succ = R.cube_reorientation_reward(c("cube_opos"), c("cube_oq"), c("cube_tpos"), c("cube_tq"),
                                              c("cube_actions"), R.CubeRewardParams())
    if dtype == np.float64:
        assert np.array_equal(succ.cpu().numpy(), a["cube_success"])
    assert rel_err(cr.double().cpu().numpy(), a["cube_reward"], 1e-3 if dtype == np.float32 else tol, tol) <= 1
    fr = R.franka_stack_reward(c("franka_a"), c("franka_b"), c("franka_g"), c("franka_l"), c("franka_r"),
                               R.FrankaStackParams())
    assert rel_err(fr.double().cpu().numpy(), a["franka_reward"], tol, tol) <= 1


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_remaining_reward_kernels_match_reference(dtype):
    """trifinger / ingenuity / AMP / rough ANYmal vs golden `rewards_extra`
    (reference rewards.py:115-121, 129-158, 179-197, 222-225)."""
    from paper_2108_10470_b200 import rewards as R
    _, a = load("rewards_extra")
    tol = 1e-10 if dtype == np.float64 else 2e-5
    c = lambda k: a[k].astype(dtype)  # noqa: E731
    tr = R.trifinger_reward(c("tri_cube"), c("tri_prev_cube"), c("tri_cube_quat"), c("tri_target"),
                            c("tri_target_quat"), c("tri_tip"), c("tri_prev_tip"), c("tri_tip_vel"),
                            a["tri_timestep"], R.TrifingerRewardParams())
    # the 1/(3 rot_dist + 0.01) term amplifies fp32 input rounding near rot_dist = 0
    assert rel_err(tr.double().cpu().numpy(), a["tri_reward"], 1e-3 if dtype == np.float32 else tol, tol) <= 1
    ir = R.ingenuity_reward(c("ing_pos"), c("ing_target"), c("ing_up"), c("ing_spin"))
    assert rel_err(ir.double().cpu().numpy(), a["ing_reward"], tol, tol) <= 1
    am = R.amp_imitation_reward(c("amp_d"))
    assert rel_err(am.double().cpu().numpy(), a["amp_reward"], 1e-3 if dtype == np.float32 else tol, tol) <= 1
    ro = R.anymal_reward(c("rough_lin"), c("rough_ang"), c("rough_cmd"), c("rough_qvel"), c("rough_qacc"),
                         c("rough_torques"), c("rough_arate"), c("rough_coll"), c("rough_air"),
                         R.AnymalRewardParams(), variant="rough")
    assert rel_err(ro.double().cpu().numpy(), a["rough_reward"], tol, tol) <= 1


def test_reward_edge_cases():
    """Empty batches launch nothing; AMP clips at both ends; the trifinger
    fingertip term switches off strictly after the cutoff."""
    import torch
    from paper_2108_10470_b200 import rewards as R
    assert R.amp_imitation_reward(np.zeros(0)).numel() == 0
    am = R.amp_imitation_reward(np.array([-5.0, 0.0, 1.0, 7.0])).cpu().numpy()
    ref = -np.log(1 - np.clip([-5.0, 0.0, 1.0, 7.0], 1e-4, 1 - 1e-4))
    assert np.allclose(am, ref, rtol=1e-12, atol=0)
    p = R.TrifingerRewardParams(w_og=0.0, w_fo=1.0, w_fv=0.0)
    z = np.zeros((2, 3))
    tip = np.tile(np.array([[[1.0, 0, 0]]]), (2, 1, 1))
    q = np.tile([0, 0, 0, 1.0], (2, 1))
    r = R.trifinger_reward(z, z, q, z, q, tip, 0.5 * tip, np.zeros((2, 1, 3)),
                           np.array([p.fingertip_term_cutoff, p.fingertip_term_cutoff + 1]), p)
    assert torch.allclose(r.cpu(), torch.tensor([0.5, 0.0], dtype=torch.float64))
