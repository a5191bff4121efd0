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
