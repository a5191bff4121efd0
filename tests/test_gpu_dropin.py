"""The reference's own task layer over the B200 step: the one-line swap of
INTEGRATION.md §1, run for real.

The unmodified reference package (installed under baseline/_ref by
``pip install --target baseline/_ref``) builds its
`QuadrupedEnv` / `AnymalObsEnv` (envs.py:359-565) with its own `SimBuffers`
(buffers.py:47-225) and `DomainRandomizer` (randomize.py:86-189); the only
change is the name `Scene` in `batchsim.envs` (envs.py:86-91), pointed at
`paper_2108_10470_b200.hostscene.HostScene`.  The same env over the
reference's NumPy `Scene` is the expected result:

  * fp64 device path: obs / reward within 1e-7 (1 + |ref|), done / timeout
    masks exact, for 16 control steps with a knock-down (terminations +
    auto-resets through the reference's own set_root_state / set_dof_state,
    world-frame writes) and timeouts at step 12;
  * fp32 device path: done / timeout masks exact and obs within the fp32
    contract for the first step from the bit-exact reset state.
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def renvs():
    if not os.path.isdir(os.path.join(REF, "batchsim")):
        pytest.skip("reference not installed under baseline/_ref (DESIGN.md §7)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import batchsim.envs as RE
    return RE


def _rollout(RE, name, scene_cls, E=48, steps=16, randomize=False):
    orig = RE.Scene
    if scene_cls is not None:
        RE.Scene = scene_cls
    try:
        env = RE.make_env(name, num_envs=E, seed=3, episode_length=12, randomize=randomize)
    finally:
        RE.Scene = orig
    rng = np.random.default_rng(11)
    knock = np.arange(1, E, 4)
    out = []
    for t in range(steps):
        if t == 5:                                     # world-frame root writes through the reference SimBuffers
            root = env.scene.root_state.copy()
            root[knock, 2] = 0.1
            env.buffers.set_root_state(root, knock)
        o = env.step(rng.uniform(-1, 1, (E, env.act_dim)))
        out.append({"obs": o.obs.copy(), "reward": o.reward.copy(), "done": o.done.copy(),
                    "timeout": o.info["timeout"].copy(), "root": env.scene.root_state.copy()})
    return env, out


@pytest.mark.parametrize("name,randomize", [("quadruped", False), ("quadruped-anymal-obs", False),
                                            ("quadruped", True)])
def test_reference_env_over_b200_scene_fp64(renvs, name, randomize):
    from paper_2108_10470_b200.hostscene import HostScene
    _, ref = _rollout(renvs, name, None, randomize=randomize)
    env, got = _rollout(renvs, name, HostScene, randomize=randomize)
    assert isinstance(env.scene, HostScene)
    n_done = 0
    for t, (r, g) in enumerate(zip(ref, got)):
        assert np.array_equal(r["done"], g["done"]), t
        assert np.array_equal(r["timeout"], g["timeout"]), t
        for k in ("obs", "reward", "root"):
            err = np.abs(g[k] - r[k]).max() / (1 + np.abs(r[k]).max())
            assert err <= 1e-7, (t, k, err)
        n_done += int(r["done"].sum())
    assert n_done >= 48          # knock-down terminations + the step-12 timeouts exercised


def test_reference_env_over_b200_scene_fp32(renvs):
    import functools

    from paper_2108_10470_b200.hostscene import HostScene
    _, ref = _rollout(renvs, "quadruped", None, steps=13)
    _, got = _rollout(renvs, "quadruped", functools.partial(HostScene, precision="fp32"), steps=13)
    for t, (r, g) in enumerate(zip(ref, got)):
        assert np.array_equal(r["done"], g["done"]), t
        assert np.array_equal(r["timeout"], g["timeout"]), t
    d = np.abs(got[0]["obs"] - ref[0]["obs"]) / (1e-4 + 1e-4 * np.abs(ref[0]["obs"]))
    assert (d <= 1).mean() >= 0.999 and d.max() <= 10, (float((d <= 1).mean()), float(d.max()))


def test_world_frame_writes_land_in_world_frame(renvs):
    """A reference-protocol caller writes world-frame `pos` (test_physics.py:123
    style); after FK the device's env-local state is that position minus the
    env origin, and the host view reads it back in world frame."""
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.hostscene import HostScene
    s = HostScene([M.quadruped()], 8)
    B = s.bodies_per_env
    target = s.env_origins[3] + np.array([0.25, -0.5, 1.5])
    s.pos[3 * B] = target
    s.forward_kinematics(env_mask=np.eye(8, dtype=bool)[3], actors={0})
    assert np.allclose(s.root_state[3, 0:3], target, atol=1e-12)
    local = s.dev.body_q[3 * B, 0:3].double().cpu().numpy()
    assert np.allclose(local, target - s.env_origins[3], atol=1e-12)
