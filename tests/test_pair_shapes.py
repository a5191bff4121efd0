"""Box / capsule pair contacts (shape_pairs="all"; not in the reference,
SURVEY.md 8(f) 2 -- parity unpinned): the slot generation rules, and the
step kernel's body compiled for the host (fp64) against the float64 C
oracle's independent narrow phase, teacher forced, on authored scenes."""

import shutil

import numpy as np
import pytest

from golden_util import rel_err
from pair_scenes import SCENES, oracle_trace


def test_pair_slot_rules():
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.layout import PAIR_CC, PAIR_PB, PAIR_PC, PAIR_SS, SceneLayout
    from pair_scenes import capsule
    sph, box, cap = M.free_sphere(), M.free_box(), capsule("c", 1.0, 0.05, 0.2)
    cases = {(sph, sph): [PAIR_SS], (sph, box): [PAIR_PB], (box, sph): [PAIR_PB], (sph, cap): [PAIR_PC],
             (cap, cap): [PAIR_CC], (cap, box): [PAIR_PB] * 2 + [PAIR_PC] * 8, (box, box): [PAIR_PB] * 16}
    for (m1, m2), kinds in cases.items():
        L = SceneLayout([m1, m2], shape_pairs="all")
        assert L.pair_kind.tolist() == kinds
        R = SceneLayout([m1, m2])                      # the reference's set: spheres only
        assert R.pair_kind.tolist() == ([PAIR_SS] if kinds == [PAIR_SS] else [])
    L = SceneLayout([box, box], shape_pairs="all")
    assert np.allclose(np.abs(L.pair_off[:8, 0]), 0.1) and np.allclose(L.pair_ext[:, :3], 0.1)
    with pytest.raises(ValueError):
        SceneLayout([box, box], shape_pairs="boxes")


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="needs nvcc as host compiler")
@pytest.mark.parametrize("name", sorted(SCENES))
def test_host_build_matches_oracle(name):
    from hostkernel.hk import HostKernel
    from paper_2108_10470_b200.layout import SceneLayout
    models, p, meta, arr = oracle_trace(name)
    E = meta["num_envs"]
    L = SceneLayout(models, True, "all")
    hk = HostKernel(L, E, p, arr["param_env_origins"], fp64=True)
    B = L.bodies_per_env
    be = np.repeat(np.arange(E), B)
    org = arr["param_env_origins"]
    for t in range(meta["steps"]):
        hk.arr["body_q"][...] = np.concatenate([arr["in_pos"][t] - org[be], arr["in_quat"][t], arr["in_linvel"][t],
                                                arr["in_angvel"][t]], 1)
        hk.arr["friction_anchor"][...] = arr["in__friction_anchor"][t] - org[None]
        for k in ("dof_state", "ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
                  "ctrl_body_torque", "dof_mode", "nonfinite"):
            hk.arr[k][...] = arr[f"in_{k}"][t]
        hk.step()
        for k in ("body_state", "net_contact"):
            assert rel_err(hk.arr[k], arr[f"out_{k}"][t], 1e-8, 1e-8) <= 1, (name, t, k)
    # the scene really exercises its pair slots
    assert np.abs(arr["out_net_contact"]).sum() > 0
