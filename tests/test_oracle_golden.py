"""Pin the CPU oracle (oracle/bso.c) to the reference's own outputs.

The fixtures were produced by running the reference `batchsim` itself
(tests/golden/make_golden.py).  Both sides are float64, so agreement is
expected to ~1e-9 (LAPACK gesv vs. the oracle's elimination differ only in
rounding)."""

import numpy as np
import pytest

from golden_util import (OUTPUTS, build_models, load, load_params, load_state,
                         physics_cases, sim_params)
from oracle.oracle import OracleScene

TOL = 1e-8


def _close(a, b, tol=TOL):
    """max |a-b| / (1 + |b|): absolute near 0, relative for large values."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    both_nan = np.isnan(a) & np.isnan(b)
    diff = np.where(both_nan, 0.0, np.abs(a - b) / (1.0 + np.abs(np.nan_to_num(b))))
    return np.nanmax(diff) if diff.size else 0.0


@pytest.mark.parametrize("case", physics_cases())
def test_oracle_teacher_forced(case):
    meta, arr = load(case)
    s = OracleScene(build_models(meta), meta["num_envs"], sim_params(meta),
                    spacing=meta["spacing"], ground=meta["ground"],
                    env_origins=arr["param_env_origins"])
    load_params(s, arr)
    for t in range(meta["steps"]):
        load_state(s, arr, t)
        s.step()
        for k in OUTPUTS:
            got, want = getattr(s, k), arr[f"out_{k}"][t]
            if k == "nonfinite":
                assert np.array_equal(got, want), (case, t, k)
                continue
            assert np.array_equal(np.isnan(got), np.isnan(want)), (case, t, k)
            assert _close(got, want) < TOL, (case, t, k, _close(got, want))


@pytest.mark.parametrize("case", [c for c in physics_cases() if c != "quadruped_nan"])
def test_oracle_free_rollout(case):
    meta, arr = load(case)
    s = OracleScene(build_models(meta), meta["num_envs"], sim_params(meta),
                    spacing=meta["spacing"], ground=meta["ground"],
                    env_origins=arr["param_env_origins"])
    load_params(s, arr)
    load_state(s, arr, 0)
    ctrl = ("ctrl_dof_force", "ctrl_dof_pos_target", "ctrl_dof_vel_target", "ctrl_body_force",
            "ctrl_body_torque", "dof_mode")
    for t in range(meta["steps"]):
        load_state(s, arr, t, ctrl)
        s.step()
    for k in ("pos", "quat", "linvel", "angvel", "dof_state", "net_contact"):
        assert _close(getattr(s, k), arr[f"out_{k}"][-1]) < 1e-7, (case, k)


@pytest.mark.parametrize("case", physics_cases())
def test_oracle_contact_list_matches_collide(case):
    """Active candidates in (slot, env) order == reference collide() list."""
    meta, arr = load(case)
    s = OracleScene(build_models(meta), meta["num_envs"], sim_params(meta),
                    spacing=meta["spacing"], ground=meta["ground"],
                    env_origins=arr["param_env_origins"])
    load_params(s, arr)
    s.pos[:] = arr["final_pos"]
    s.quat[:] = arr["final_quat"]
    act, depth, point, normal = s.contact_geometry()
    B, E = s.bodies_per_env, s.num_envs
    P = s.layout.planes_per_env
    ba, bb = [], []
    for i in range(P + s.layout.pairs_per_env):
        for e in range(E):
            if not act[i * E + e]:
                continue
            if i < P:
                ba.append(-1)
                bb.append(e * B + s.layout.plane_body[i])
            else:
                a, b = s.layout.pair_body[i - P]
                ba.append(e * B + a)
                bb.append(e * B + b)
    assert np.array_equal(ba, arr["collide_body_a"]), case
    assert np.array_equal(bb, arr["collide_body_b"]), case
    sel = act
    assert _close(depth[sel], arr["collide_depth"]) < 1e-12
    assert _close(point[sel], arr["collide_point"]) < 1e-12
    assert _close(normal[sel], arr["collide_normal"]) < 1e-12
