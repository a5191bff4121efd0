"""The oracle's test instrumentation (oracle/bso.h `margin`, `limit_jitter*`)
observes without perturbing: decision margins recorded, outputs bit-identical
to an uninstrumented run; limit re-decisions only touch joints within the
knife-edge tolerance (a zero tolerance changes nothing).  CPU only."""

import numpy as np

from oracle.tasks import OracleEnv


def _run(E=16, steps=6, margin=False, jitter=None):
    env = OracleEnv("humanoid", E, seed=3, episode_length=100)
    s = env.scene
    rng = np.random.default_rng(5)
    out, margins = [], []
    for t in range(steps):
        a = rng.uniform(-1, 1, (E, env.act_dim))
        if margin:
            s.decision_margin = np.full((E, 4), np.inf)
        s.limit_jitter = jitter
        obs, reward, done, _ = env.step(a)
        if margin:
            margins.append(s.decision_margin.copy())
            s.decision_margin = None
        out.append(np.concatenate([s.pos.ravel(), s.linvel.ravel(), s.angvel.ravel(), obs.ravel()]))
    return np.stack(out), margins


def test_margins_observe_without_perturbing():
    base, _ = _run()
    inst, margins = _run(margin=True)
    assert np.array_equal(base, inst)
    m = np.stack(margins)
    assert np.all(m >= 0)
    assert np.isfinite(m[:, :, 0]).all()          # every humanoid env evaluates its limit rows
    assert np.isfinite(m[:, :, 1]).all()          # and its ground slots


def test_limit_jitter_zero_tolerance_is_identity():
    base, _ = _run()
    same, _ = _run(jitter=(7, 0.0))
    assert np.array_equal(base, same)


def test_limit_jitter_changes_only_envs_within_tolerance():
    """With a tolerance between the envs' smallest limit margins, the envs
    whose every limit decision sat farther away step bit-identically and the
    others move (the re-decision perturbs q, hence the limit bias)."""
    E, steps = 16, 6
    base, margins = _run(E, steps, margin=True)
    m = np.stack(margins)[:, :, 0].min(axis=0)             # per env, relative to max(1, |limit|)
    tol = float(np.median(m))
    jit, _ = _run(E, steps, jitter=(7, tol))
    env = OracleEnv("humanoid", E, seed=3, episode_length=100)
    B, O = env.scene.bodies_per_env, env.obs_dim
    n3 = E * B * 3

    def env_cols(e):
        cols = [np.arange(k * n3 + e * B * 3, k * n3 + (e + 1) * B * 3) for k in range(3)]
        return np.concatenate(cols + [np.arange(3 * n3 + e * O, 3 * n3 + (e + 1) * O)])

    far, near = np.nonzero(m > tol)[0], np.nonzero(m < tol)[0]
    assert len(far) and len(near)
    for e in far:
        assert np.array_equal(base[:, env_cols(e)], jit[:, env_cols(e)]), e
    assert any(not np.array_equal(base[:, env_cols(e)], jit[:, env_cols(e)]) for e in near)
