"""The CUDA step's per-env code (csrc/bsim_step.cuh) compiled for the host and
checked against the float64 oracle, fp64 and fp32, on every golden case.

This runs on CPU-only machines (it only needs nvcc as a host compiler), so the
kernel arithmetic is validated before any GPU time is spent.  It is a test of
the kernel source, not a product path: the product always launches the
sm_100a kernels.
"""

import shutil

import numpy as np
import pytest

from golden_util import PARAMS, build_models, load, physics_cases, rel_err, sim_params

pytestmark = pytest.mark.skipif(shutil.which("nvcc") is None, reason="needs nvcc as host compiler")


def _local(arr, t, E, B, key):
    org = arr["param_env_origins"]
    be = np.repeat(np.arange(E), B)
    bq = np.concatenate([arr[f"{key}pos"][t] - org[be], arr[f"{key}quat"][t],
                         arr[f"{key}linvel"][t], arr[f"{key}angvel"][t]], 1)
    return bq, arr[f"{key}_friction_anchor"][t] - org[None]


def _host(case, fp64, specialize=True):
    from hostkernel.hk import HostKernel
    from paper_2108_10470_b200.layout import SceneLayout
    meta, arr = load(case)
    L = SceneLayout(build_models(meta), meta["ground"])
    hk = HostKernel(L, meta["num_envs"], sim_params(meta), arr["param_env_origins"], fp64=fp64,
                    specialize=specialize)
    for k in PARAMS:
        hk.arr[k][...] = arr[f"param_{k}"]
    return meta, arr, L, hk


def _load(hk, arr, t, E, B):
    bq, fa = _local(arr, t, E, B, "in_")
    hk.arr["body_q"][...] = bq
    hk.arr["friction_anchor"][...] = fa
    for k in ("dof_state", "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target",
              "ctrl_body_force", "ctrl_body_torque", "dof_mode", "nonfinite"):
        hk.arr[k][...] = arr[f"in_{k}"][t]


@pytest.mark.parametrize("specialize", [True, False])
@pytest.mark.parametrize("case", physics_cases())
def test_host_build_fp64_matches_reference(case, specialize):
    meta, arr, L, hk = _host(case, True, specialize)
    E, B = meta["num_envs"], L.bodies_per_env
    for t in range(meta["steps"]):
        _load(hk, arr, t, E, B)
        hk.step()
        bad = np.repeat(arr["out_nonfinite"][t], B)
        for k in ("body_state", "net_contact"):
            assert rel_err(hk.arr[k][~bad], arr[f"out_{k}"][t][~bad], 1e-8, 1e-8) <= 1, (case, t, k)
        assert rel_err(hk.arr["dof_state"], arr["out_dof_state"][t], 1e-6, 1e-6) <= 1, (case, t)


@pytest.mark.parametrize("case", ["quadruped_walk", "kitchen_sink", "cartpole_force"])
def test_host_build_fused_substeps(case):
    """n_substeps=2 in one call == the reference's two consecutive steps."""
    meta, arr, L, hk = _host(case, True)
    E, B = meta["num_envs"], L.bodies_per_env
    _load(hk, arr, 0, E, B)
    # the controls of step 0 and 1 must match for a fused comparison
    for k in ("ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
              "ctrl_body_torque"):
        if not np.array_equal(arr[f"in_{k}"][0], arr[f"in_{k}"][1]):
            pytest.skip("controls change between recorded steps")
    hk.step(2)
    assert rel_err(hk.arr["body_state"], arr["out_body_state"][1], 1e-8, 1e-8) <= 1
