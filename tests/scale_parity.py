"""fp32 / fp64 parity of the CUDA env step at BASELINE.json scale (4096 envs)
against the float64 reference, per quantity.

Chain of evidence:
  reference EnvBatch (4096 envs, 20 free control steps, knock-downs, timeouts)
    -> tests/golden/scale_*_4096.npz (post-step state + outputs of a 1/32 env
       sample every step, done / timeout masks of ALL envs every step)
    -> the oracle (oracle/tasks.py over oracle/bso.c) re-runs the same 4096
       envs free and must match the sample at 1e-7 and the full masks exactly
       (tests/test_oracle_golden.py) -- it then stands in for the reference
       on every env
    -> the CUDA path, two ways:
       * teacher forced: before each step the oracle's full pre-step state is
         loaded, one control step runs, every output is compared;
       * free rollout: the CUDA env runs the 20 steps from construction on its
         own and the per-step error and the first divergence step are reported.

Errors are reported per quantity with the north-star contract
|gpu - ref| <= 1e-4 + 1e-4 |ref| ("scaled" error <= 1): the fraction of
elements inside it, the 99.9th percentile and max of the absolute error and
the max scaled error.  Positions are compared env-local (the canonical GPU
state; world positions at 4096 envs reach 250 m, where the fp32 ulp alone is
1.5e-5 m).  Used by tests/test_gpu_scale_parity.py and tools/parity_table.py.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from golden_util import load

CASES = {"quadruped": "scale_ant_4096", "quadruped-anymal-obs": "scale_anymal_4096",
         "humanoid": "scale_humanoid_4096"}
QUANTITIES = ("root_state", "body_state", "dof_state", "net_contact", "sensor_forces", "dof_force", "obs",
              "reward")
ATOL = RTOL = 1e-4


def oracle_trace(task, threads=None):
    """Free-run the oracle env over the fixture's schedule; returns (meta,
    fixture arrays, list of per-step {"pre": ..., "post": ...})."""
    from oracle.tasks import OracleEnv
    meta, arr = load(CASES[task])
    E = meta["num_envs"]
    env = OracleEnv(task, E, seed=meta["seed"], episode_length=meta["episode_length"],
                    threads=threads or os.cpu_count() or 1)
    s = env.scene
    knock = np.arange(1, E, 4)
    rng = np.random.default_rng(0)
    steps = []
    for t in range(meta["steps"]):
        a = rng.uniform(-1.0, 1.0, (E, env.act_dim))
        if t == meta["knock_step"]:
            root = env.local_root()[knock]
            root[:, 2] = knock_z(meta) - s.env_origins[knock, 2]
            env.set_root_state(root, knock)
        pre = {"pos": s.pos.copy(), "quat": s.quat.copy(), "linvel": s.linvel.copy(), "angvel": s.angvel.copy(),
               "anchor": s._friction_anchor.copy(), "dof_state": s.dof_state.copy(),
               "root_state": s.root_state.copy(), "sensor_forces": s.sensor_forces.copy(),
               "dof_force": s.dof_force.copy(), "episode_steps": env.episode_steps.copy(),
               "reset_count": env.reset_count.copy(), "potentials": env.potentials.copy(),
               "commands": env.commands.copy(), "actions": a}
        s.decision_margin = np.full((E, 4), np.inf)
        obs, reward, done, info = env.step(a)
        margin, s.decision_margin = s.decision_margin, None
        post = {"obs": obs, "reward": reward, "done": done, "timeout": info["timeout"], "margin": margin,
                "body_local": local_body(s.pos, s.quat, s.linvel, s.angvel, s.env_origins, s.bodies_per_env),
                "dof_state": s.dof_state.copy(), "net_contact": s.net_contact.copy(),
                "sensor_forces": s.sensor_forces.copy(), "dof_force": s.dof_force.copy(),
                "anchor": s._friction_anchor.copy(), "reset_count": env.reset_count.copy()}
        steps.append({"pre": pre, "post": post})
    return meta, arr, steps


def knock_z(meta):
    """The world z the fixture knocks every 4th env to (meta "knock" ends in
    "world z = <z>"): 0.1 for the quadrupeds, 0.5 for the humanoid, both
    below the task's termination height."""
    return float(meta["knock"].rsplit("=", 1)[1])


def local_body(pos, quat, linvel, angvel, origins, B):
    E = len(origins)
    be = np.repeat(np.arange(E), B)
    return np.concatenate([pos - origins[be], quat, linvel, angvel], 1)


def make_gpu_env(task, meta, precision):
    from paper_2108_10470_b200.envs import make_env
    return make_env(task, num_envs=meta["num_envs"], seed=meta["seed"], episode_length=meta["episode_length"],
                    precision=precision)


def load_pre(env, pre):
    """The oracle's pre-step state into the CUDA env (env-local positions)."""
    s = env.scene
    E, B = s.num_envs, s.bodies_per_env
    org = s.env_origins_host
    dt = s.dtype
    s.body_q.copy_(torch.as_tensor(local_body(pre["pos"], pre["quat"], pre["linvel"], pre["angvel"], org, B),
                                   dtype=dt))
    s._friction_anchor.copy_(torch.as_tensor(pre["anchor"] - org[None], dtype=dt))
    for k in ("dof_state", "root_state", "sensor_forces", "dof_force"):
        getattr(s, k).copy_(torch.as_tensor(pre[k], dtype=dt))
    env.episode_steps.copy_(torch.as_tensor(pre["episode_steps"].astype(np.int32)))
    env.reset_count.copy_(torch.as_tensor(pre["reset_count"].astype(np.int32)))
    env.potentials.copy_(torch.as_tensor(pre["potentials"], dtype=env.potentials.dtype))
    env.commands.copy_(torch.as_tensor(pre["commands"], dtype=env.commands.dtype))


def gpu_post(env, out):
    s = env.scene
    B = s.bodies_per_env
    bq = s.body_q.double().cpu().numpy()
    return {"obs": out.obs.double().cpu().numpy(), "reward": out.reward.double().cpu().numpy(),
            "done": out.done.cpu().numpy(), "timeout": out.info["timeout"].cpu().numpy(),
            "body_state": bq, "root_state": bq[::B], "dof_state": s.dof_state.double().cpu().numpy(),
            "net_contact": s.net_contact.double().cpu().numpy(),
            "sensor_forces": s.sensor_forces.double().cpu().numpy(),
            "dof_force": s.dof_force.double().cpu().numpy(),
            "anchor": s._friction_anchor.double().cpu().numpy(),
            "reset_count": env.reset_count.cpu().numpy()}


def ref_post(post, B):
    d = dict(post)
    d["body_state"] = post["body_local"]
    d["root_state"] = post["body_local"][::B]
    return d


# Vector quantities are judged relative to the magnitude of the VECTOR they
# belong to (|g_i - r_i| <= 1e-4 + 1e-4 |r_vec|): a 268 N contact force with a
# 0.3 N tangential component carries rounding proportional to 268 N in every
# component (the friction-basis rotation of its impulses), so an element-wise
# relative bound on the 0.3 N component measures the basis, not the solver.
# Groups of consecutive columns per row; quantities not listed are scalar.
VECTOR_GROUPS = {"root_state": (3, 4, 3, 3), "body_state": (3, 4, 3, 3), "net_contact": (3,),
                 "sensor_forces": (3, 3)}


def _magnitude(q, r):
    """|r| per element: the norm of its vector group (VECTOR_GROUPS), else |r_i|."""
    groups = VECTOR_GROUPS.get(q)
    r = np.asarray(r, float)
    if groups is None or r.ndim != 2 or r.shape[1] != sum(groups):
        return np.abs(r)
    out = np.empty_like(r)
    c = 0
    for n in groups:
        out[:, c:c + n] = np.linalg.norm(r[:, c:c + n], axis=1, keepdims=True)
        c += n
    return out


def quantity_errors(g, r, q=None):
    """{max_abs, p999_abs, max_scaled, frac_within} of |g - r| vs 1e-4 + 1e-4 |r|
    (|r| per VECTOR_GROUPS for vector quantities; `*_elem` = element-wise |r_i|)."""
    mag = _magnitude(q, r).ravel()
    g = np.asarray(g, float).ravel()
    r = np.asarray(r, float).ravel()
    d = np.abs(g - r)
    sc = d / (ATOL + RTOL * mag)
    se = d / (ATOL + RTOL * np.abs(r))
    return {"max_abs": float(d.max()), "p999_abs": float(np.quantile(d, 0.999)), "max_scaled": float(sc.max()),
            "frac_within": float(np.mean(sc <= 1.0)), "max_scaled_elem": float(se.max()),
            "frac_within_elem": float(np.mean(se <= 1.0)), "n": int(d.size)}


def compare(gp, rp):
    return {q: quantity_errors(gp[q], rp[q], q) for q in QUANTITIES}


def masks_equal(gp, rp):
    """done / timeout / reset counts exact; friction-anchor presence (NaN) pattern."""
    return {"done": bool(np.array_equal(gp["done"], rp["done"])),
            "timeout": bool(np.array_equal(gp["timeout"], rp["timeout"])),
            "reset_count": bool(np.array_equal(gp["reset_count"], rp["reset_count"])),
            "anchor_mismatch": int(np.sum(np.isnan(gp["anchor"][..., 0]) != np.isnan(rp["anchor"][..., 0])))}


def teacher_forced(task, precision, trace=None):
    """Per step: (errors per quantity, mask equality) of one CUDA control step
    from the oracle's pre-step state."""
    meta, arr, steps = trace if trace is not None else oracle_trace(task)
    env = make_gpu_env(task, meta, precision)
    B = env.scene.bodies_per_env
    res = []
    for st in steps:
        load_pre(env, st["pre"])
        out = env.step(torch.as_tensor(st["pre"]["actions"], dtype=env.scene.dtype))
        gp = gpu_post(env, out)
        rp = ref_post(st["post"], B)
        res.append({"errors": compare(gp, rp), "masks": masks_equal(gp, rp), "gpu": gp, "ref": rp})
    env.close()
    return meta, arr, res


def free_rollout(task, precision, trace=None):
    """The CUDA env free from construction over the fixture's schedule."""
    meta, arr, steps = trace if trace is not None else oracle_trace(task)
    env = make_gpu_env(task, meta, precision)
    s = env.scene
    B = s.bodies_per_env
    knock = np.arange(1, meta["num_envs"], 4)
    res = []
    for t, st in enumerate(steps):
        if t == meta["knock_step"]:
            root = s.root_state.clone()
            root[knock, 2] = knock_z(meta)
            env.buffers.set_root_state(root, knock)
        out = env.step(torch.as_tensor(st["pre"]["actions"], dtype=s.dtype))
        gp = gpu_post(env, out)
        rp = ref_post(st["post"], B)
        res.append({"errors": compare(gp, rp), "masks": masks_equal(gp, rp), "gpu": gp, "ref": rp})
    env.close()
    return meta, arr, res


def sample_dims(arr):
    """(bodies, dofs, sensors) per env, from the fixture's sampled rows."""
    n = len(arr["sample"])
    return len(arr["body_state"][0]) // n, len(arr["dof_state"][0]) // n, len(arr["sensor_forces"][0]) // n


def sample_vs_reference(meta, arr, gp, t, B, D, S):
    """The CUDA outputs of the fixture's env sample vs the reference itself."""
    idx = arr["sample"]
    rb = (idx[:, None] * B + np.arange(B)).ravel()
    rd = (idx[:, None] * D + np.arange(D)).ravel()
    rs = (idx[:, None] * S + np.arange(S)).ravel()
    org = np.repeat(arr["env_origins"], B, axis=0)
    body = arr["body_state"][t].copy()
    body[:, 0:3] -= org
    ref = {"obs": arr["obs"][t], "reward": arr["reward"][t], "body_state": body, "root_state": body[::B],
           "dof_state": arr["dof_state"][t], "net_contact": arr["net_contact"][t],
           "sensor_forces": arr["sensor_forces"][t], "dof_force": arr["dof_force"][t]}
    g = {"obs": gp["obs"][idx], "reward": gp["reward"][idx], "body_state": gp["body_state"][rb],
         "root_state": gp["body_state"][rb][::B], "dof_state": gp["dof_state"][rd],
         "net_contact": gp["net_contact"][rb], "sensor_forces": gp["sensor_forces"][rs],
         "dof_force": gp["dof_force"][rd]}
    return {q: quantity_errors(g[q], ref[q], q) for q in QUANTITIES}


def _r32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def _perturbed_runs(task, trace, transforms, threads=None):
    """Per transform, per step: the float64 oracle's post-step outputs (the
    ref_post layout) from the TRANSFORMED pre-state (transform(x) applied to
    env-local positions, orientations, velocities, DOF state, anchors,
    commands and actions)."""
    from oracle.tasks import OracleEnv
    meta, arr, steps = trace
    E = meta["num_envs"]
    env = OracleEnv(task, E, seed=meta["seed"], episode_length=meta["episode_length"],
                    threads=threads or os.cpu_count() or 1)
    s = env.scene
    B = s.bodies_per_env
    org = np.repeat(s.env_origins, B, axis=0)
    out = []
    for tf in transforms:
        runs = []
        for t, st in enumerate(steps):
            if isinstance(tf, _LimitJitter):      # exact pre-state, knife-edge limits re-decided
                s.limit_jitter = (tf.seed * 1000 + t + 1, LIMIT_MARGIN)
            else:
                s.limit_jitter = None
            pre = st["pre"]
            s.pos[:] = org + tf(pre["pos"] - org)
            for k in ("quat", "linvel", "angvel"):
                getattr(s, k)[:] = tf(pre[k])
            s._friction_anchor[:] = s.env_origins[None] + tf(pre["anchor"] - s.env_origins[None])
            for k in ("dof_state", "root_state", "sensor_forces", "dof_force"):
                getattr(s, k)[:] = tf(pre[k])
            env.episode_steps[:] = pre["episode_steps"]
            env.reset_count[:] = pre["reset_count"]
            env.potentials[:] = pre["potentials"]
            env.commands[:] = tf(pre["commands"])
            obs, reward, done, info = env.step(tf(pre["actions"]))
            post = {"obs": obs, "reward": reward, "done": done, "timeout": info["timeout"],
                    "body_local": local_body(s.pos, s.quat, s.linvel, s.angvel, s.env_origins, B),
                    "dof_state": s.dof_state.copy(), "net_contact": s.net_contact.copy(),
                    "sensor_forces": s.sensor_forces.copy(), "dof_force": s.dof_force.copy()}
            runs.append(ref_post(post, B))
        out.append(runs)
    return out


class _LimitJitter:
    """Identity transform; the oracle re-decides every joint-limit activation
    within LIMIT_MARGIN of its threshold at random (bso.h limit_jitter)."""

    def __init__(self, seed):
        self.seed = seed

    def __call__(self, x):
        return x


def _jitter(seed):
    """x (1 + u 2^-24), u uniform in [-1, 1]: an fp32-sized relative perturbation."""
    rng = np.random.default_rng(seed)

    def tf(x):
        x = np.asarray(x, np.float64)
        return x * (1.0 + rng.uniform(-1.0, 1.0, x.shape) * 2.0 ** -24)
    return tf


def input_rounding_floor(task, trace=None, threads=None):
    """The fp32 conditioning floor, per step and quantity: the float64 oracle
    stepped from the fp32-ROUNDED pre-state and actions (env-local positions,
    as the CUDA path stores them) vs the oracle from the exact pre-state.  No
    fp32 arithmetic is involved, so any fp32 implementation of the reference
    algorithm inherits at least this error."""
    trace = trace if trace is not None else oracle_trace(task)
    runs = _perturbed_runs(task, trace, [_r32], threads)[0]
    return [compare(r, ref_post(st["post"], _bodies(trace))) for r, st in zip(runs, trace[2])]


def _bodies(trace):
    meta, _, steps = trace
    return len(steps[0]["post"]["body_local"]) // meta["num_envs"]


def sensitivity(task, trace=None, seeds=(1, 2), threads=None):
    """Per step and quantity, the element-wise max |oracle(perturbed) -
    oracle(exact)| over the fp32 rounding of the pre-state and len(seeds)
    random fp32-sized relative perturbations of it: how far the reference
    algorithm itself moves each output under input noise of the size fp32
    storage makes.  An element whose GPU error is within a few times this is
    ill-conditioned at fp32 (a friction stick / slip, limit or contact
    activation decided within rounding), not mis-computed."""
    trace = trace if trace is not None else oracle_trace(task)
    B = _bodies(trace)
    runs = _perturbed_runs(task, trace, [_r32] + [_jitter(sd) for sd in seeds], threads)
    out = []
    for t, st in enumerate(trace[2]):
        ref = ref_post(st["post"], B)
        out.append({q: np.max([np.abs(np.asarray(r[t][q], float) - np.asarray(ref[q], float)) for r in runs], axis=0)
                    for q in QUANTITIES})
    return out


# A joint-limit activation decided within 8 fp32 ulps of the joint angle
# (|q - limit| <= 2^-21 max(1, |limit|) in some pass of the reference's step)
# is a coin flip for an fp32 state -- the joint angle stored in fp32 and
# recomputed from fp32 orientations is uncertain by several ulps -- and a
# limit row that engages in one precision and not in the other changes the
# joint's velocity by the whole approach rate.  Input jitter (sensitivity())
# rarely flips these: TGS drives an engaged joint onto its limit, so the
# later passes' q sit within ulps of it whatever the input noise.
# limit_sensitivity() re-decides them at random instead.
LIMIT_MARGIN = 2.0 ** -21


def limit_sensitivity(task, trace=None, seeds=(1, 2, 3, 4), threads=None):
    """Per step and quantity, the element-wise max |oracle(knife-edge limits
    re-decided) - oracle(exact)| over len(seeds) random re-decisions: how far
    the reference itself moves when the joint-limit activations it decided
    within LIMIT_MARGIN (8 fp32 ulps of the joint angle) go the other way, as
    they may in any fp32 implementation."""
    trace = trace if trace is not None else oracle_trace(task)
    B = _bodies(trace)
    runs = _perturbed_runs(task, trace, [_LimitJitter(sd) for sd in seeds], threads)
    out = []
    for t, st in enumerate(trace[2]):
        ref = ref_post(st["post"], B)
        out.append({q: np.max([np.abs(np.asarray(r[t][q], float) - np.asarray(ref[q], float)) for r in runs], axis=0)
                    for q in QUANTITIES})
    return out


# Contact and sensor forces are impulses / dt summed in a Gauss-Seidel sweep:
# every impulse of an env is computed from velocities that its other impulses
# moved, so its rounding scales with the env's LARGEST force, not its own (a
# 6 mN grazing contact of the ANYmal base next to 80 N foot contacts).  An
# element beyond the bound relative to its own vector but within it relative
# to its env's largest force vector of that quantity is "within the env's
# force resolution".
FORCE_QUANTITIES = ("net_contact", "sensor_forces")


def _env_force_scale(q, r2, E):
    """Per row: the largest vector norm of quantity q in the row's env."""
    k = len(r2) // E
    groups = VECTOR_GROUPS[q]
    norms = np.zeros(len(r2))
    c = 0
    for n in groups:
        norms = np.maximum(norms, np.linalg.norm(r2[:, c:c + n], axis=1))
        c += n
    return np.repeat(norms.reshape(E, k).max(axis=1), k)


def excused(gp, rp, sens, q, bound_scaled=10.0, factor=0.1, lsens=None):
    """Elements of quantity q beyond `bound_scaled` x (1e-4 + 1e-4 |ref|)
    (|ref| per VECTOR_GROUPS) split into (excused, unexplained): an element is
    excused when the reference's own output moves by at least `factor` x the
    GPU deviation under fp32-sized input noise (`sens`, sensitivity()) or
    when its knife-edge joint-limit decisions are re-decided (`lsens`,
    limit_sensitivity()), or -- forces -- when it is within the bound relative
    to its env's largest force (FORCE_QUANTITIES)."""
    a, b, c, unexplained = excused_split(gp, rp, sens, q, bound_scaled, factor, lsens)
    return a + b + c, unexplained


def excused_split(gp, rp, sens, q, bound_scaled=10.0, factor=0.1, lsens=None):
    """(ill by input noise, ill by knife-edge limits, within the env's force
    resolution, unexplained) element counts."""
    r = np.asarray(rp[q], float)
    r2 = r.reshape(len(r), -1) if r.ndim > 1 else r.reshape(-1, 1)
    d = np.abs(np.asarray(gp[q], float).reshape(r2.shape) - r2)
    sc = d / (ATOL + RTOL * _magnitude(q, r2))
    over = sc > bound_scaled
    ill = over & (np.asarray(sens[q], float).reshape(r2.shape) >= factor * d)
    knife = np.zeros_like(over)
    if lsens is not None:
        knife = over & ~ill & (np.asarray(lsens[q], float).reshape(r2.shape) >= factor * d)
    coupled = np.zeros_like(over)
    if q in FORCE_QUANTITIES and "reward" in rp:
        scale = _env_force_scale(q, r2, len(rp["reward"]))
        coupled = over & ~ill & ~knife & (d <= bound_scaled * (ATOL + RTOL * scale)[:, None])
    return int(ill.sum()), int(knife.sum()), int(coupled.sum()), int((over & ~ill & ~knife & ~coupled).sum())
