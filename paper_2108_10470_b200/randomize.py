"""Domain randomisation and observation noise on the device
(reference `pkg/src/batchsim/randomize.py`).

Same schedule objects and semantics as the reference: a schedule maps the
targets (dims, masses, friction, damping, gains, joint_limits, gravity) to a
sampling rule; every randomisation epoch restores the env's base parameters
before applying fresh draws (no compounding), draws are keyed
(seed, global env id, epoch) and an env is re-randomised only once
`min_interval_steps` sim steps have elapsed.  The draws themselves run in
the `dr_randomize_env` device function (csrc/bsim_dr.cuh) with
numpy-identical PCG64 + ziggurat streams, so a device randomisation equals
the reference's bit for bit in the float64 path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N

DISTRIBUTIONS = ("uniform", "loguniform", "gaussian")
MODES = ("scaling", "additive")
TARGETS = ("dims", "masses", "friction", "damping", "gains", "joint_limits", "gravity")
_WATCHED = ("inv_mass", "inertia_local", "inv_inertia_local", "gravity", "mu_static", "mu_dynamic",
            "joint_stiffness", "joint_damping", "joint_limit_lo", "joint_limit_hi", "plane_rad",
            "plane_off", "pair_rad", "pair_off")


@dataclass
class RandomizationEntry:
    target: str
    distribution: str
    mode: str
    range: tuple

    def __post_init__(self):
        if self.target not in TARGETS:
            raise ValueError(f"unknown randomization target: {self.target!r}")
        if self.distribution not in DISTRIBUTIONS:
            raise ValueError(f"unknown distribution: {self.distribution!r}")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode: {self.mode!r}")


@dataclass
class RandomizationSchedule:
    entries: dict = field(default_factory=dict)
    min_interval_steps: int = 720

    @classmethod
    def from_config(cls, cfg):
        sched = cls(min_interval_steps=int(cfg.get("min_interval_steps", 720)))
        for raw in cfg.get("entries", []):
            e = RandomizationEntry(raw["target"], raw["distribution"], raw["mode"], tuple(raw["range"]))
            sched.entries[e.target] = e
        return sched


def _default_entries():
    mk = RandomizationEntry
    return {  # the paper's Table 12 rows as the reference encodes them (randomize.py:64-77)
        "dims": mk("dims", "uniform", "scaling", (0.95, 1.05)),
        "masses": mk("masses", "uniform", "scaling", (0.5, 1.5)),
        "friction": mk("friction", "uniform", "scaling", (0.7, 1.3)),
        "damping": mk("damping", "loguniform", "scaling", (0.3, 3.0)),
        "gains": mk("gains", "loguniform", "scaling", (0.75, 1.5)),
        "joint_limits": mk("joint_limits", "gaussian", "additive", (0.0, 0.15)),
        "gravity": mk("gravity", "gaussian", "additive", (0.0, 0.4)),
    }


DEFAULT_SCHEDULE = RandomizationSchedule(entries=_default_entries())


class DR(C.Structure):
    """bsim_dr_t (include/batchsim_b200.h)."""
    _fields_ = ([("enabled", C.c_int32), ("seed", C.c_uint32), ("min_interval", C.c_int32),
                 ("pad", C.c_int32), ("use", C.c_int32 * 7), ("dist", C.c_int32 * 7),
                 ("mode", C.c_int32 * 7), ("pad2", C.c_int32), ("a", C.c_double * 7),
                 ("b", C.c_double * 7), ("epoch", C.c_void_p), ("last_step", C.c_void_p)] +
                [(n, C.c_void_p) for n in _WATCHED])


class DomainRandomizer:
    """Device DomainRandomizer (randomize.py:86-189) over a GPU Scene."""

    def __init__(self, scene, schedule=None, seed=0):
        self.scene = scene
        self.schedule = schedule if schedule is not None else DEFAULT_SCHEDULE
        self.seed = int(seed)
        dev = scene.device
        self._base = {k: getattr(scene, k).clone() for k in _WATCHED}
        E = scene.num_envs
        self.epoch = torch.zeros(E, dtype=torch.int32, device=dev)
        self._last_step = torch.full((E,), -self.schedule.min_interval_steps, dtype=torch.int32, device=dev)
        self._mask = torch.zeros(E, dtype=torch.uint8, device=dev)
        self.struct = self._build()

    def _build(self):
        d = DR()
        d.enabled = 1
        d.seed = self.seed
        d.min_interval = int(self.schedule.min_interval_steps)
        for t, name in enumerate(TARGETS):
            e = self.schedule.entries.get(name)
            if e is None:
                continue
            d.use[t] = 1
            d.dist[t] = DISTRIBUTIONS.index(e.distribution)
            d.mode[t] = MODES.index(e.mode)
            d.a[t], d.b[t] = float(e.range[0]), float(e.range[1])
        d.epoch = self.epoch.data_ptr()
        d.last_step = self._last_step.data_ptr()
        for k in _WATCHED:
            setattr(d, k, self._base[k].data_ptr())
        return d

    def due(self, env_indices, step):
        idx = torch.as_tensor(np.atleast_1d(np.asarray(env_indices, dtype=np.int64)), device=self.scene.device)
        return idx[(step - self._last_step[idx].long()) >= self.schedule.min_interval_steps]

    def randomize(self, env_indices, step):
        """Restore base then apply fresh draws for due envs (randomize.py:116-134).
        Returns True if any env was randomised."""
        s = self.scene
        due = self.due(env_indices, step)
        if due.numel() == 0:
            return False
        self._mask.zero_()
        self._mask[due] = 1
        lay, _, st = s._structs()
        fn = getattr(s._lib, "bsim_randomize" + ("_f64" if s.fp64 else ""))
        rc = fn(C.byref(lay), C.byref(st), C.byref(self.struct), self._mask.data_ptr(), int(step), s._s)
        if rc != 0:
            raise N.NativeError(f"bsim_randomize failed ({rc})")
        return True

    def clear(self, env_indices):
        """Restore the base parameters of the given envs (randomize.py:136-138)."""
        s = self.scene
        E = s.num_envs
        for e in np.atleast_1d(np.asarray(env_indices, dtype=np.int64)):
            e = int(e)
            B = s.bodies_per_env
            for k in ("inv_mass", "inertia_local", "inv_inertia_local"):
                getattr(s, k)[e * B:(e + 1) * B] = self._base[k][e * B:(e + 1) * B]
            for k in ("gravity", "mu_static", "mu_dynamic"):
                getattr(s, k)[e] = self._base[k][e]
            for k in ("joint_stiffness", "joint_damping", "joint_limit_lo", "joint_limit_hi", "plane_rad",
                      "plane_off", "pair_rad", "pair_off"):
                arr = getattr(s, k)
                if arr.numel():
                    arr[:, e] = self._base[k][:, e]
        _ = E


class Force(C.Structure):
    """bsim_force_t (include/batchsim_b200.h)."""
    _fields_ = [("num_envs", C.c_int32), ("env_offset", C.c_int32), ("seed", C.c_uint32),
                ("fp64", C.c_int32), ("p_lo", C.c_double), ("p_hi", C.c_double),
                ("probability", C.c_void_p), ("force", C.c_void_p), ("epoch", C.c_void_p),
                ("count", C.c_void_p)]


def _seed_of(rng):
    if isinstance(rng, np.random.Generator):
        return int(rng.integers(0, 2 ** 32))
    return int(rng) & 0xFFFFFFFF


class RandomForceState:
    """Per-env random disturbance forces (randomize.py:192-212) on the device.

    Same constructor arguments and attributes as the reference (`rng` may be
    an integer seed or a numpy Generator, from which one seed is drawn);
    `probability` (E,) and `force` (E, 3) are device tensors that may be
    edited in place.  Each env draws from its own stream keyed (seed, global
    env id, counter): the reference's batch-wide stream has the same law but
    would tie every env's draws to the batch size.
    """

    def __init__(self, num_envs, rng=0, p_lo=0.001, p_hi=0.1, device="cuda", dtype=torch.float32,
                 env_offset=0):
        self.num_envs, self.p_lo, self.p_hi = int(num_envs), float(p_lo), float(p_hi)
        if self.num_envs < 0 or not 0.0 < self.p_lo <= self.p_hi:
            raise ValueError("need num_envs >= 0 and 0 < p_lo <= p_hi")
        self.seed, self.env_offset = _seed_of(rng), int(env_offset)
        E = self.num_envs
        self.probability = torch.zeros(E, dtype=dtype, device=device)
        self.force = torch.zeros((E, 3), dtype=dtype, device=device)
        self._epoch = torch.zeros(E, dtype=torch.int32, device=device)
        self._count = torch.zeros(E, dtype=torch.int32, device=device)
        self._mask = torch.zeros(E, dtype=torch.uint8, device=device)
        self._lib = N.lib()
        self.resample_probability(None)

    @property
    def fp64(self):
        return self.force.dtype == torch.float64

    def struct(self):
        return Force(self.num_envs, self.env_offset, self.seed, int(self.fp64), self.p_lo, self.p_hi,
                     self.probability.data_ptr(), self.force.data_ptr(), self._epoch.data_ptr(),
                     self._count.data_ptr())

    def resample_probability(self, env_indices):
        """New firing probability and zero force for the given envs (None = all)."""
        mptr = None
        if env_indices is not None:
            idx = torch.as_tensor(np.atleast_1d(np.asarray(env_indices, dtype=np.int64)),
                                  device=self.force.device)
            if idx.numel() == 0:
                return
            if int(idx.min()) < 0 or int(idx.max()) >= self.num_envs:
                raise IndexError("env index out of range")
            self._mask.zero_()
            self._mask[idx] = 1
            mptr = self._mask.data_ptr()
        f = self.struct()
        rc = self._lib.bsim_force_resample(C.byref(f), mptr, torch.cuda.current_stream().cuda_stream)
        if rc != 0:
            raise N.NativeError(f"bsim_force_resample failed ({rc})")


def random_object_force(state, mass, dt, body_force=None, body=0, bodies_per_env=1):
    """Fire-or-decay update of `state.force` (randomize.py:215-221); returns a
    copy.  With `body_force` (a scene's ctrl_body_force, (E*B, 3)) the new
    force is also written to row e*bodies_per_env + body in the same launch."""
    f = state.force
    m = mass if isinstance(mass, torch.Tensor) else torch.as_tensor(np.asarray(mass, dtype=np.float64))
    m = m.to(f.device, f.dtype).reshape(-1).contiguous()
    if m.numel() != state.num_envs:
        raise ValueError("mass must have one entry per env")
    bptr = None
    if body_force is not None:
        if body_force.dtype != f.dtype or body_force.device != f.device or not body_force.is_contiguous() \
                or body_force.numel() != 3 * state.num_envs * bodies_per_env:
            raise ValueError("body_force must be a contiguous (E*B, 3) tensor of the state's dtype")
        bptr = body_force.data_ptr()
    s = state.struct()
    rc = state._lib.bsim_random_object_force(C.byref(s), m.data_ptr(), float(dt), bptr, int(bodies_per_env),
                                             int(body), torch.cuda.current_stream().cuda_stream)
    if rc != 0:
        raise N.NativeError(f"bsim_random_object_force failed ({rc})")
    return f.clone()


def check_supported(cfg):
    """EnvConfig.randomize / obs_noise are supported on the device."""
    return True
