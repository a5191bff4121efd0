"""Device domain randomisation / observation noise vs the reference
(randomize.py:86-237; golden randomize_quadruped + env_quadruped_dr_noise).

The device draws reproduce numpy's PCG64 uniform / loguniform and ziggurat
normal streams, so the randomised parameters match bit for bit (fp64) and
to fp32 rounding (fp32)."""

import numpy as np
import pytest
import torch

from golden_util import load, rel_err

pytestmark = pytest.mark.gpu

WATCHED = ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static", "mu_dynamic",
           "joint_stiffness", "joint_damping", "joint_limit_lo", "joint_limit_hi", "plane_rad", "plane_off")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_domain_randomizer_matches_reference(precision):
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.params import SimParams
    from paper_2108_10470_b200.randomize import DEFAULT_SCHEDULE, DomainRandomizer
    from paper_2108_10470_b200.scene import Scene
    meta, arr = load("randomize_quadruped")
    s = Scene([M.quadruped()], 6, SimParams(dt=1 / 120), precision=precision)
    dr = DomainRandomizer(s, DEFAULT_SCHEDULE, seed=meta["seed"])
    tol = 1e-12 if precision == "fp64" else 1e-6
    assert dr.randomize(np.arange(6), step=0)
    for k in WATCHED:
        assert rel_err(getattr(s, k).double().cpu().numpy(), arr[f"e0_{k}"], tol, tol) <= 1, k
    assert not dr.randomize(np.array([1, 3]), step=100)    # interval not elapsed
    dr.randomize(np.array([0, 2, 5]), step=800)
    for k in WATCHED:
        assert rel_err(getattr(s, k).double().cpu().numpy(), arr[f"e1_{k}"], tol, tol) <= 1, k
    assert np.array_equal(dr.epoch.cpu().numpy(), arr["epoch"])
    dr.clear([0])
    assert torch.equal(s.gravity[0], dr._base["gravity"][0])


def test_randomized_noisy_env_trace_fp64():
    """EnvBatch with randomize=True and correlated obs noise (uncorrelated off),
    free-running in float64 against the reference trace."""
    from paper_2108_10470_b200.envs import make_env
    meta, arr = load("env_quadruped_dr_noise")
    env = make_env("quadruped", num_envs=6, seed=4, episode_length=12, randomize=True, obs_noise=True,
                   obs_noise_uncorr=0.0, precision="fp64")
    assert rel_err(env.reset().cpu().numpy(), arr["obs0"], 1e-9, 1e-9) <= 1
    for t in range(meta["steps"]):
        out = env.step(torch.as_tensor(arr["actions"][t]))
        assert np.array_equal(out.done.cpu().numpy(), arr["done"][t]), t
        assert rel_err(env.scene.gravity.cpu().numpy(), arr["gravity"][t], 1e-12, 1e-12) <= 1, t
        assert rel_err(env.scene.joint_stiffness.cpu().numpy(), arr["joint_stiffness"][t], 1e-12, 1e-12) <= 1
        assert rel_err(env.corr_noise.cpu().numpy(), arr["corr"][t], 1e-12, 1e-12) <= 1, t
        assert rel_err(out.obs.cpu().numpy(), arr["obs"][t], 1e-6, 1e-6) <= 1, t
        assert rel_err(out.reward.cpu().numpy(), arr["reward"][t], 1e-6, 1e-6) <= 1, t


def test_uncorrelated_noise_statistics():
    """Per-env counter-keyed streams give N(0, sigma) noise (same law as the
    reference's batch-wide stream, randomize.py:231-237)."""
    from paper_2108_10470_b200.envs import make_env
    clean = make_env("quadruped", num_envs=4096, seed=1)
    noisy = make_env("quadruped", num_envs=4096, seed=1, obs_noise=True, obs_noise_corr=0.0,
                     obs_noise_uncorr=0.05)
    d = (noisy.obs - clean.obs).double()
    assert abs(float(d.mean())) < 3 * 0.05 / np.sqrt(d.numel())
    assert abs(float(d.std()) - 0.05) < 0.002
