"""Tensor-API facade on the GPU (reference buffers.py + tests/test_buffers.py).

Indexed setters are checked against the reference's own results
(tests/golden buffers_quadruped: set_root_state then set_dof_state on actor
subsets, including forward kinematics and quaternion renormalisation), and
the complement-rows-untouched contract is checked bitwise.
"""

import numpy as np
import pytest
import torch

from golden_util import load, rel_err

pytestmark = pytest.mark.gpu


def _scene(E=6, precision="fp64"):
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.params import SimParams
    from paper_2108_10470_b200.scene import Scene
    return Scene([M.quadruped()], E, SimParams(dt=1 / 120), precision=precision)


def _load_state(s, arr, prefix):
    E, B = s.num_envs, s.bodies_per_env
    org = arr["env_origins"][np.repeat(np.arange(E), B)]
    bq = np.concatenate([arr[f"{prefix}_pos"] - org, arr[f"{prefix}_quat"], arr[f"{prefix}_linvel"],
                         arr[f"{prefix}_angvel"]], 1)
    s.body_q.copy_(torch.as_tensor(bq, dtype=s.dtype))
    for k in ("root_state", "body_state", "dof_state"):
        getattr(s, k).copy_(torch.as_tensor(arr[f"{prefix}_{k}"], dtype=s.dtype))


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_indexed_setters_match_reference(precision):
    from paper_2108_10470_b200.buffers import SimBuffers
    meta, arr = load("buffers_quadruped")
    s = _scene(meta["num_envs"], precision)
    buf = SimBuffers(s)
    _load_state(s, arr, "before")
    tol = 1e-9 if precision == "fp64" else 1e-5
    buf.set_root_state(torch.as_tensor(arr["root_values"]), arr["idx_root"])
    for k in ("root_state", "body_state", "dof_state"):
        assert rel_err(getattr(s, k).double().cpu().numpy(), arr[f"mid_{k}"], tol, tol) <= 1, k
    buf.set_dof_state(arr["dof_values"], arr["idx_dof"])
    for k in ("root_state", "body_state", "dof_state"):
        assert rel_err(getattr(s, k).double().cpu().numpy(), arr[f"after_{k}"], tol, tol) <= 1, k


def test_acquire_aliases_canonical_storage():
    from paper_2108_10470_b200.buffers import SimBuffers, UnknownKind
    s = _scene(2)
    buf = SimBuffers(s)
    assert buf.acquire("root_state") is s.root_state
    assert buf.acquire("dof_state") is s.dof_state
    assert buf.acquire("controls")["dof_pos_target"] is s.ctrl_dof_pos_target
    with pytest.raises(UnknownKind):
        buf.acquire("bogus")


def test_error_contract():
    from paper_2108_10470_b200.buffers import (IndexOutOfRange, ModeMismatch, NonFiniteWrite,
                                               ShapeMismatch, SimBuffers, UnknownKind)
    s = _scene(2)
    buf = SimBuffers(s)
    with pytest.raises(ShapeMismatch):
        buf.set_root_state(np.zeros((3, 13)))
    with pytest.raises(IndexOutOfRange):
        buf.set_root_state(s.root_state.clone(), [s.num_actors])
    bad = s.root_state.clone()
    bad[0, 7] = float("nan")
    with pytest.raises(NonFiniteWrite):
        buf.set_root_state(bad, [0])
    deg = s.root_state.clone()
    deg[1, 3:7] = 0
    with pytest.raises(NonFiniteWrite):
        buf.set_root_state(deg, [1])
    with pytest.raises(ModeMismatch):   # position-mode drives (buffers.py:209-218)
        buf.submit_controls("dof_force", np.zeros(s.num_dofs))
    with pytest.raises(UnknownKind):
        buf.submit_controls("bogus", np.zeros(1))


def test_indexed_isolation_random_sets():
    """tests/test_buffers.py:115-152: complement rows are byte-identical."""
    from paper_2108_10470_b200.buffers import SimBuffers
    s = _scene(8, "fp32")
    buf = SimBuffers(s)
    rng = np.random.default_rng(0)
    s.pos[:, 2] += 0.37
    s.forward_kinematics()
    for _ in range(5):
        s.ctrl_dof_pos_target.copy_(torch.as_tensor(rng.uniform(-0.3, 0.3, s.num_dofs)))
        s.step()
    B, D = s.bodies_per_env, s.dofs_per_env
    for trial in range(30):
        k = int(rng.integers(1, 5))
        envs = rng.choice(8, size=k, replace=False)
        keep_b = np.ones(s.num_bodies, bool)
        keep_d = np.ones(s.num_dofs, bool)
        for e in envs:
            keep_b[e * B:(e + 1) * B] = False
            keep_d[e * D:(e + 1) * D] = False
        before = (s.body_q.cpu().numpy()[keep_b].tobytes(), s.dof_state.cpu().numpy()[keep_d].tobytes(),
                  s.body_state.cpu().numpy()[keep_b].tobytes())
        if trial % 2 == 0:
            root = s.root_state.clone()
            root[envs, 0:3] = torch.as_tensor(s.env_origins_host[envs] + rng.uniform([-1, -1, 0.3], [1, 1, 0.6], (k, 3)),
                                              dtype=root.dtype, device=root.device)
            buf.set_root_state(root, envs)
        else:
            dof = s.dof_state.clone().reshape(8, -1, 2)
            dof[envs] = torch.as_tensor(rng.uniform(-0.5, 0.5, (k, D, 2)), dtype=dof.dtype, device=dof.device)
            buf.set_dof_state(dof.reshape(-1, 2), envs)
        after = (s.body_q.cpu().numpy()[keep_b].tobytes(), s.dof_state.cpu().numpy()[keep_d].tobytes(),
                 s.body_state.cpu().numpy()[keep_b].tobytes())
        assert before == after, trial


def test_tensor_api_roundtrip():
    from paper_2108_10470_b200.tensor_api import TensorAPI
    s = _scene(4, "fp32")
    gym = TensorAPI(s)
    root = gym.acquire_actor_root_state_tensor()
    assert root is s.root_state
    gym.set_dof_position_target_tensor(torch.full((s.num_dofs,), 0.2))
    assert torch.all(s.ctrl_dof_pos_target == 0.2)
    z0 = root[:, 2].clone()
    gym.simulate(2)
    gym.fetch_results()
    assert not torch.equal(z0, root[:, 2])
