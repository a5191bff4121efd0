"""Pin the CPU oracle (oracle/bso.c) to the reference's own outputs.

The fixtures were produced by running the reference `batchsim` itself
(tests/golden/make_golden.py).  Both sides are float64, so agreement is
expected to ~1e-9 (LAPACK gesv vs. the oracle's elimination differ only in
rounding)."""

import os

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


ENV_CASES = [("quadruped", "env_quadruped", 0.1, "potentials"),
             ("quadruped-anymal-obs", "env_quadruped_anymal_obs", 0.1, "commands"),
             ("humanoid", "env_humanoid", 0.5, "potentials")]


@pytest.mark.parametrize("task,fixture,knock_z,extra", ENV_CASES)
def test_oracle_env_free_running_matches_reference(task, fixture, knock_z, extra):
    """The oracle task layer (oracle/tasks.py) over the C physics, FREE running
    from construction through the reference's whole env trace (its explicit
    second reset, the knock-over of env 2 at t = 5, terminations, timeouts at
    episode_length and the auto-resets): obs / reward / done / timeout and
    the env-layer state agree with the reference EnvBatch at 1e-7, done and
    timeout masks and reset counts exactly."""
    from oracle.tasks import OracleEnv
    meta, arr = load(fixture)
    env = OracleEnv(task, meta["num_envs"], seed=meta["seed"], episode_length=meta["episode_length"])
    assert _close(env.scene.env_origins, arr["env_origins"]) < 1e-12
    obs0 = env.reset()
    assert _close(obs0, arr["obs0"]) < 1e-9
    for t in range(meta["steps"]):
        if t == 5:
            root = env.local_root()[[2]]
            root[0, 2] = knock_z - env.scene.env_origins[2, 2]
            env.set_root_state(root, np.array([2]))
        assert np.array_equal(env.reset_count, arr["reset_count"][t]), t
        assert np.array_equal(env.episode_steps, arr["episode_steps"][t]), t
        assert _close(getattr(env, extra), arr["extra_before"][t]) < 1e-7, (t, extra)
        obs, reward, done, info = env.step(arr["actions"][t])
        assert np.array_equal(done, arr["done"][t]), t
        assert np.array_equal(info["timeout"], arr["timeout"][t]), t
        assert _close(obs, arr["obs"][t]) < 1e-7, (t, "obs", _close(obs, arr["obs"][t]))
        assert _close(reward, arr["reward"][t]) < 1e-7, (t, "reward")
        assert _close(env.scene.ctrl_dof_pos_target, arr["ctrl_dof_pos_target"][t]) < 1e-12, t


@pytest.mark.parametrize("task", ["quadruped", "quadruped-anymal-obs", "humanoid"])
def test_oracle_env_at_4096_envs_matches_reference(task):
    """BASELINE scale: the oracle env free running over the reference's 4096-env
    trace (tests/golden/make_scale_golden.py: 20 control steps, a quarter of
    the envs knocked down at step 5, every env timing out at step 12):
    done / timeout masks of ALL envs exact at every step, the reference's
    1/32 env sample (post-step state, obs, reward, env-layer state) at 1e-7.
    The oracle then stands in for the reference on every env of the CUDA
    parity tests (tests/test_gpu_scale_parity.py)."""
    import scale_parity as SP
    meta, arr, steps = SP.oracle_trace(task, threads=os.cpu_count() or 1)
    idx = arr["sample"]
    B = SP.sample_dims(arr)[0]
    rb = (idx[:, None] * B + np.arange(B)).ravel()
    org = np.repeat(arr["env_origins"], B, axis=0)
    for t, st in enumerate(steps):
        p = st["post"]
        assert np.array_equal(p["done"], arr["done_all"][t]), t
        assert np.array_equal(p["timeout"], arr["timeout_all"][t]), t
        assert np.array_equal(p["reset_count"][idx], arr["reset_count"][t]), t
        body = arr["body_state"][t].copy()
        body[:, 0:3] -= org
        assert _close(p["body_local"][rb], body) < 1e-7, (t, "body")
        assert _close(p["obs"][idx], arr["obs"][t]) < 1e-7, (t, "obs")
        assert _close(p["reward"][idx], arr["reward"][t]) < 1e-7, (t, "reward")
        assert _close(p["net_contact"][rb], arr["net_contact"][t]) < 1e-7, (t, "net_contact")
        assert _close(p["anchor"][:, idx], arr["friction_anchor"][t]) < 1e-7, (t, "anchors")
    assert arr["done_all"].sum() >= 4096          # terminations and timeouts both exercised
