"""Every form of the Gauss-Seidel row schedule runs the reference's
sequential sweep (physics.py:760-775) on the GPU: with each mode forced
(BSIM_SCHED_MODE = asap / phased / joints; the launcher then runs the
scheduled step-kernel instantiation) a scene steps like the same scene on
the one-lane sequential sweep (BSIM_SCHED_MODE = none, the sequential
instantiation), fp64 to rounding.  Rows of one stage touch disjoint bodies,
so only the instruction mix of the two kernels differs.  The cost model's
own pick is covered by every other GPU test; this pins the forms it does
not pick today (tests/test_sweep_schedule.py checks the schedules
themselves on the CPU)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

_TRACES = {}


def _trace(name):
    import pair_scenes as PS
    if name not in _TRACES:
        _TRACES[name] = PS.oracle_trace(name)
    return _TRACES[name]


def _scene(name, mode, monkeypatch):
    from golden_util import load_gpu_state
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.scene import Scene
    monkeypatch.setenv("BSIM_SCHED_MODE", mode)
    if name == "humanoid":
        s = Scene([M.humanoid()], 64, precision="fp64")
        s.pos[:, 2] += 1.0
        s.forward_kinematics()
        return s
    if name == "kitchen_sink":      # the default-CTA kernel: every joint kind, tendons, sphere pairs
        from golden_util import build_models, load, sim_params
        meta, arr = load("kitchen_sink")
        s = Scene(build_models(meta), meta["num_envs"], sim_params(meta), precision="fp64",
                  env_origins=arr["param_env_origins"])
        load_gpu_state(s, arr, 0)
        return s
    models, p, meta, arr = _trace(name)
    s = Scene(models, meta["num_envs"], p, precision="fp64", shape_pairs="all", env_origins=arr["param_env_origins"])
    load_gpu_state(s, arr, 0)
    return s


@pytest.mark.parametrize("mode", ["asap", "phased", "joints"])
@pytest.mark.parametrize("name", ["humanoid", "shadow_hand_cube", "franka_cube_stack", "kitchen_sink"])
def test_forced_schedule_equals_sequential_sweep(name, mode, monkeypatch):
    a = _scene(name, mode, monkeypatch)
    b = _scene(name, "none", monkeypatch)
    assert a.layout.sweep_schedule()[0] == mode and b.layout.sweep_schedule()[0] is None
    g = np.random.default_rng(3)
    for _ in range(16):
        act = torch.as_tensor(g.uniform(-1, 1, (a.num_envs, a.dofs_per_env)), device="cuda")
        a.step(2, actions=act, action_scale=0.3)
        b.step(2, actions=act, action_scale=0.3)
    qa, qb = a.body_q.cpu().numpy(), b.body_q.cpu().numpy()
    assert np.isfinite(qa).all()
    assert np.abs(qa - qb).max() <= 1e-9 * (1 + np.abs(qb).max()), np.abs(qa - qb).max()
    na, nb = a.net_contact.cpu().numpy(), b.net_contact.cpu().numpy()
    assert np.abs(na - nb).max() <= 1e-7 * (1 + np.abs(nb).max())
