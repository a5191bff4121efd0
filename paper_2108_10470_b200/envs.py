"""Vectorised RL tasks on the GPU scene (reference `pkg/src/batchsim/envs.py`).

Same classes, config, registry and step/reset contract as the reference
`EnvBatch` (envs.py:73-205): actions are clipped to [-1, 1] and scaled into
position targets, the physics runs `decimation` sim steps, then reward, done
(termination | timeout | poisoned), observation and auto-reset are produced
-- here by two launches per control step:

1. ``bsim_step``: the fused action mapping + all decimation substeps;
2. ``bsim_task_step``: one thread per env computes reward / done / obs and,
   for finished envs, draws the reset state with numpy-identical PCG64
   streams keyed (seed, global env id, reset count), runs forward kinematics
   and writes the post-reset observation.

Outputs are device tensors that alias persistent buffers (zero-copy; clone a
result to keep it across steps).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace
from typing import NamedTuple

import numpy as np
import torch

from . import _native as N
from . import models as M
from .buffers import SimBuffers
from .layout import MODE_POSITION
from .params import SimParams
from .randomize import DEFAULT_SCHEDULE, DR, DomainRandomizer
from .scene import Scene

ALL = None
TASK_QUADRUPED, TASK_ANYMAL, TASK_HUMANOID, TASK_CUBE, TASK_STACK = 1, 2, 3, 4, 5


@dataclass
class EnvConfig:
    """Reference EnvConfig (envs.py:38-63) plus the B200 knobs."""
    num_envs: int = 16
    seed: int = 0
    sim_dt: float = 1.0 / 120.0
    control_dt: float = 1.0 / 60.0
    episode_length: int = 1000
    workers: int = 1
    randomize: bool = False
    obs_noise: bool = False
    obs_noise_uncorr: float = 0.002
    obs_noise_corr: float = 0.001
    extra: dict = field(default_factory=dict)
    precision: str = "fp32"
    device: str | None = None
    env_offset: int = 0           # global id of env 0 (multi-GPU sharding)
    total_envs: int | None = None

    def validate(self):
        if self.num_envs < 1:
            raise ValueError("num_envs must be >= 1")
        ratio = self.control_dt / self.sim_dt
        if abs(ratio - round(ratio)) > 1e-9 or round(ratio) < 1:
            raise ValueError("control_dt must be a positive integer multiple of sim_dt")
        if not 0 <= self.seed < 2 ** 32:
            raise ValueError("seed must fit in 32 bits")
        return self

    @property
    def decimation(self):
        return int(round(self.control_dt / self.sim_dt))


class StepOutput(NamedTuple):
    obs: torch.Tensor
    reward: torch.Tensor
    done: torch.Tensor
    info: dict


class Task(C.Structure):
    """bsim_task_t (include/batchsim_b200.h)."""
    _fields_ = [("kind", C.c_int32), ("obs_dim", C.c_int32), ("act_dim", C.c_int32),
                ("episode_length", C.c_int32), ("seed", C.c_uint32), ("obs_noise", C.c_int32),
                ("control_dt", C.c_double), ("rest_height", C.c_double),
                ("obs_noise_uncorr", C.c_double), ("obs_noise_corr", C.c_double),
                ("step_count", C.c_int64)] + [
        (n, C.c_void_p) for n in ("obs", "reward", "done", "timeout", "poisoned", "episode_steps",
                                  "reset_count", "actions", "potentials", "commands", "dof_lower",
                                  "dof_upper", "corr_noise", "noise_count")] + [("dr", DR),
                                                                                ("termination_height", C.c_double),
                                                                                ("step_count_dev", C.c_void_p),
                                                                                ("goals", C.c_void_p)]


def dof_limits(model):
    """Per-DOF (lower, upper); unlimited DOFs get +-inf (envs.py:28-35)."""
    lo, hi = [], []
    for j in model.joints:
        for _ in range(j.dof_count):
            lo.append(j.limits[0] if j.limits else -np.inf)
            hi.append(j.limits[1] if j.limits else np.inf)
    return np.asarray(lo, float), np.asarray(hi, float)


class EnvBatch:
    """Base: GPU scene construction, fused decimated stepping, auto-reset."""

    name = "base"
    obs_dim = 0
    act_dim = 0
    action_scale = 1.0
    task_kind = 0
    rest_height = 0.0
    termination_height = 0.26     # LocomotionRewardParams.termination_height (rewards.py:25)

    def __init__(self, config: EnvConfig):
        self.config = cfg = config.validate()
        E = cfg.num_envs
        self.model = self._model()
        self.scene = self.sim = Scene(self._models(), E, self._sim_params(), device=cfg.device,
                                      precision=cfg.precision, env_offset=cfg.env_offset,
                                      total_envs=cfg.total_envs, **self._scene_kwargs())
        self.buffers = SimBuffers(self.scene)
        s = self.scene
        dev, dt = s.device, s.dtype
        self.obs = torch.zeros((E, self.obs_dim), dtype=dt, device=dev)
        self.reward = torch.zeros(E, dtype=dt, device=dev)
        self.done = torch.zeros(E, dtype=torch.bool, device=dev)
        self.timeout = torch.zeros(E, dtype=torch.bool, device=dev)
        self.poisoned = torch.zeros(E, dtype=torch.bool, device=dev)
        self.episode_steps = torch.zeros(E, dtype=torch.int32, device=dev)
        self.reset_count = torch.zeros(E, dtype=torch.int32, device=dev)
        self.actions = torch.zeros((E, self.act_dim), dtype=dt, device=dev)
        self.potentials = torch.zeros(E, dtype=torch.float64, device=dev)   # float64 in both precisions
        self.commands = torch.zeros((E, 3), dtype=dt, device=dev)
        lo, hi = dof_limits(self.model)
        self.dof_lower = torch.as_tensor(lo, dtype=dt, device=dev)
        self.dof_upper = torch.as_tensor(hi, dtype=dt, device=dev)
        self._mask = torch.zeros(E, dtype=torch.uint8, device=dev)
        self.corr_noise = torch.zeros((E, self.obs_dim), dtype=dt, device=dev)
        self.noise_count = torch.zeros(E, dtype=torch.int32, device=dev)
        self.goals = (torch.zeros((E, 8), dtype=dt, device=dev) if self.task_kind in (TASK_CUBE, TASK_STACK)
                      else None)
        self._setup()
        # domain randomisation (envs.py:94-96): snapshot after scene construction
        self._graph = None
        self.randomizer = (DomainRandomizer(self.scene, DEFAULT_SCHEDULE, seed=cfg.seed)
                           if cfg.randomize else None)
        self._task = Task(self.task_kind, self.obs_dim, self.act_dim, cfg.episode_length, cfg.seed,
                          int(cfg.obs_noise), cfg.control_dt, self.rest_height,
                          float(cfg.obs_noise_uncorr), float(cfg.obs_noise_corr), 0,
                          *(t.data_ptr() for t in (self.obs, self.reward, self.done, self.timeout,
                                                   self.poisoned, self.episode_steps, self.reset_count,
                                                   self.actions, self.potentials, self.commands,
                                                   self.dof_lower, self.dof_upper, self.corr_noise,
                                                   self.noise_count)),
                          self.randomizer.struct if self.randomizer is not None else DR(),
                          float(self.termination_height), None,
                          self.goals.data_ptr() if self.goals is not None else None)
        self.reset()

    # ------------------------------------------------------------ hooks
    def _model(self):
        raise NotImplementedError

    def _models(self):
        return [self.model]

    def _scene_kwargs(self):
        return {}

    def _setup(self):
        """Task buffers / fixed poses to set before the first reset."""

    def _sim_params(self):
        return SimParams(dt=self.config.sim_dt)

    # ------------------------------------------------------------ helpers
    def _call(self, name, *args):
        self._task.step_count = int(self.scene.step_count)
        self._task.step_count_dev = None
        lib = self.scene._lib
        fn = getattr(lib, name + ("_f64" if self.scene.fp64 else ""))
        lay, _, st = self.scene._structs()
        rc = fn(C.byref(lay), C.byref(st), C.byref(self._task), *args)
        if rc != 0:
            raise N.NativeError(f"{name} failed ({rc}): {lib.bsim_task_last_error().decode()}")

    def local_root(self):
        """Root states with the env origins removed (envs.py:135-139)."""
        root = self.scene.root_state.clone()
        root[:, 0:3] -= self.scene.env_origins.repeat_interleave(self.scene.actors_per_env, 0)
        return root

    def dof_view(self):
        return self.scene.dof_state.reshape(self.config.num_envs, -1, 2)

    # ------------------------------------------------------------ API
    @N.on_scene_device
    def reset(self, env_indices=ALL):
        """Reset all envs (None) or the given ones; returns the full obs."""
        E = self.config.num_envs
        mptr = None
        if env_indices is not None:
            idx = torch.as_tensor(np.atleast_1d(np.asarray(env_indices, dtype=np.int64))
                                  if not isinstance(env_indices, torch.Tensor) else env_indices,
                                  device=self.scene.device).reshape(-1).long()
            if idx.numel() == 0:
                return self.obs
            if int(idx.min()) < 0 or int(idx.max()) >= E:
                raise IndexError("env index out of range")
            self._mask.zero_()
            self._mask[idx] = 1
            mptr = self._mask.data_ptr()
        self._call("bsim_task_reset", mptr, self.scene._s)
        return self.obs

    @N.on_scene_device
    def step(self, actions) -> StepOutput:
        cfg = self.config
        a = actions if isinstance(actions, torch.Tensor) else torch.as_tensor(np.asarray(actions, dtype=np.float64))
        if tuple(a.shape) != (cfg.num_envs, self.act_dim):
            raise ValueError(f"actions must have shape ({cfg.num_envs}, {self.act_dim})")
        a = a.to(self.scene.device, self.scene.dtype)
        if self._graph is not None and self._graph_gen != self.scene._struct_gen:
            self.capture_graph()       # set_params() changed the structs baked into the graph
        if self._graph is not None:
            self._graph_in.copy_(a)
            self._graph.replay()
            self.scene.step_count += cfg.decimation
        else:
            if not a.is_contiguous():
                a = a.contiguous()
            self._step_launches(a)
        return StepOutput(self.obs, self.reward, self.done,
                          {"timeout": self.timeout, "poisoned": self.poisoned})

    # True: one launch per control step (bsim_env_step, the task tail runs in
    # the physics kernel, obs rows staged in the dead workspace and stored
    # coalesced); its ctypes argument block is built once and re-pointed per
    # call.  Measured on B200 (16384 Ant envs): device time equal to the
    # two-launch path (266 vs 265 us) and ~15 us less host time per step, so
    # it is the default; False = bsim_step then bsim_task_step.
    fused = True

    def _step_launches(self, a, graph=False):
        """The control step's launches: the fused physics + task-tail launch
        (bsim_env_step), or physics (bsim_step) then the task layer."""
        cfg = self.config
        sc = self.scene
        if graph:   # the replayed step reads / advances the device step counter
            self._step_count_dev.add_(cfg.decimation)
        if self.fused:
            lay, par, st = sc._structs()
            key = (id(lay), id(par), id(st), sc._s, graph)
            fz = self.__dict__.get("_fused_args")
            if fz is None or fz[0] != key:
                act = N.Actions(0, self.actions.data_ptr(), float(self.action_scale), MODE_POSITION, 0)
                args = (C.byref(lay), C.byref(par), C.byref(st), int(cfg.decimation), C.byref(act),
                        C.byref(self._task), sc._s)
                fz = self._fused_args = (key, act, args, sc._sfx("bsim_env_step"))
            _, act, args, fn = fz
            act.actions = a.data_ptr()
            self._task.step_count = int(sc.step_count) + cfg.decimation
            self._task.step_count_dev = self._step_count_dev.data_ptr() if graph else None
            rc = fn(*args)
            self._task.step_count_dev = None
            N.check(rc, "bsim_env_step")
            sc.step_count += cfg.decimation
            return
        sc.step(cfg.decimation, actions=a, action_scale=self.action_scale, action_mode=MODE_POSITION,
                actions_clipped=self.actions)
        if graph:
            lib = sc._lib
            fn = getattr(lib, "bsim_task_step" + ("_f64" if sc.fp64 else ""))
            lay, _, st = sc._structs()
            self._task.step_count_dev = self._step_count_dev.data_ptr()
            rc = fn(C.byref(lay), C.byref(st), C.byref(self._task), sc._s)
            self._task.step_count_dev = None
            if rc != 0:
                raise N.NativeError(f"bsim_task_step failed ({rc}): {lib.bsim_task_last_error().decode()}")
        else:
            self._call("bsim_task_step", sc._s)

    @N.on_scene_device
    def capture_graph(self, warmup=0):
        """Capture one control step (physics launch + task launch + the device
        step counter the DR interval reads) into a CUDA graph; later `step()`
        calls copy the actions into the graph's static input and replay it --
        the same launches with the same arguments as the eager path, one graph
        launch per control step.  `warmup` eager zero-action steps run first
        (they advance the envs like ordinary steps).  `release_graph()` returns
        to eager launches."""
        cfg = self.config
        dev = self.scene.device
        self._graph_in = torch.zeros((cfg.num_envs, self.act_dim), dtype=self.scene.dtype, device=dev)
        for _ in range(warmup):
            self.step(self._graph_in)
        self._step_count_dev = torch.full((1,), int(self.scene.step_count), dtype=torch.int64, device=dev)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        main, count = self.scene.stream, self.scene.step_count
        g = torch.cuda.CUDAGraph()
        object.__setattr__(self.scene, "stream", side)
        try:
            with torch.cuda.graph(g, stream=side):
                self._step_launches(self._graph_in, graph=True)
        finally:
            object.__setattr__(self.scene, "stream", main)
            self.scene.step_count = count          # capture executed nothing
        self._graph = g
        self._graph_gen = self.scene._struct_gen
        return g

    def release_graph(self):
        self._graph = None

    # ------------------------------------------------------------ host-buffer step
    # True: each chunk is one bsim_env_step_range launch (physics + task tail);
    # False: bsim_step_range then bsim_task_step_range.
    host_fused = False
    # env chunks of the host step; 0 = one per step-kernel wave
    host_chunks = 0
    # replay the host step as one captured CUDA graph (bsim_env_step_host_graph)
    host_graph = True
    # zero-copy host step (bsim_env_step_host mode 2): one fused launch on
    # the mapped pinned buffers; host_chunks / host_fused / host_graph unused.
    # Measured on B200 (16384 Ant envs, tools/host_step_bench.py): 328 us per
    # control step vs 354 us for the best pipelined-chunk schedule.
    host_zero_copy = True

    def _host_init(self):
        cfg, sc = self.config, self.scene
        E, dt = cfg.num_envs, sc.dtype
        pin = dict(pin_memory=True)
        h = {"act": torch.empty((E, self.act_dim), dtype=dt, **pin),
             "act_dev": torch.empty((E, self.act_dim), dtype=dt, device=sc.device),
             "obs": torch.empty((E, self.obs_dim), dtype=dt, **pin),
             "reward": torch.empty(E, dtype=dt, **pin),
             "done": torch.empty(E, dtype=torch.bool, **pin),
             "timeout": torch.empty(E, dtype=torch.bool, **pin),
             "poisoned": torch.empty(E, dtype=torch.bool, **pin),
             "pinned": {}, "graph": None, "graph_key": None, "eager_steps": 0,
             "count_host": torch.zeros(1, dtype=torch.int64, **pin),
             "count_dev": torch.zeros(1, dtype=torch.int64, device=sc.device)}
        self._host = h
        return h

    def host_chunk_count(self):
        """Env chunks step_host uses: host_chunks, or one per wave of the step
        kernel (bsim_step_envs_per_wave)."""
        if self.host_chunks > 0:
            return min(self.host_chunks, 16, self.config.num_envs)
        h = getattr(self, "_host", None) or self._host_init()
        if "auto_chunks" in h:
            return h["auto_chunks"]
        sc = self.scene
        wave = C.c_int32(0)
        lay, _, _ = sc._structs()
        N.check(sc._lib.bsim_step_envs_per_wave(C.byref(lay), int(sc.fp64), C.byref(wave)),
                "bsim_step_envs_per_wave")
        h["auto_chunks"] = min(16, max(1, -(-self.config.num_envs // max(1, wave.value))))
        return h["auto_chunks"]

    @N.on_scene_device
    def step_host(self, actions, sync=True) -> StepOutput:
        """EnvBatch.step with HOST arrays (the reference's numpy call,
        envs.py:178-200): actions (E, act_dim) numpy / CPU tensor in, CPU
        (pinned) obs / reward / done / info out, in one native call
        (bsim_env_step_host): the batch runs as wave-sized env chunks, each on
        its own stream once its actions are uploaded, and chunk c's outputs
        stream back over PCIe while chunk c+1 steps.  Results equal `step()`'s
        bitwise (envs are independent).  Outputs alias persistent pinned
        buffers; with sync=False they are valid once the scene stream is
        synchronised.  Pinned float actions of the scene dtype are read in
        place; anything else is staged through a pinned buffer first."""
        cfg, sc = self.config, self.scene
        h = getattr(self, "_host", None) or self._host_init()
        a = actions if isinstance(actions, torch.Tensor) else torch.from_numpy(np.asarray(actions))
        if tuple(a.shape) != (cfg.num_envs, self.act_dim):
            raise ValueError(f"actions must have shape ({cfg.num_envs}, {self.act_dim})")
        src = None
        if a.device.type == "cpu" and a.dtype == sc.dtype and a.is_contiguous():
            key = a.data_ptr()
            pinned = h["pinned"].get(key)
            if pinned is None:               # is_pinned() queries the driver: cache it per buffer
                if len(h["pinned"]) > 64:
                    h["pinned"].clear()
                pinned = h["pinned"][key] = bool(a.is_pinned())
            if pinned:
                src = a
        inflight = h.get("inflight")      # a previous sync=False step may still read h["act"] /
        if inflight is not None and (src is None or not self.host_zero_copy):   # count_host
            inflight.synchronize()
            h["inflight"] = None
        if src is None:
            src = h["act"].copy_(a)
        structs = sc._structs()
        lay, par, st = structs
        post = int(sc.step_count) + cfg.decimation
        if self.host_zero_copy:
            self._step_host_zero_copy(src, h, lay, par, st, post)
            sc.step_count += cfg.decimation
            self._host_done(h, sync)
            return StepOutput(h["obs"], h["reward"], h["done"], {"timeout": h["timeout"], "poisoned": h["poisoned"]})
        n_chunks = int(self.host_chunk_count())
        key = (sc._struct_gen, n_chunks, bool(self.host_fused))
        if self.host_graph and h["graph"] is not None and h["graph_key"] == key:
            rc = sc._lib.bsim_host_graph_launch(h["graph"], src.data_ptr(), post, sc._s)
            if rc != 0:
                raise N.NativeError(f"bsim_host_graph_launch failed ({rc}): {sc._lib.bsim_host_last_error().decode()}")
        else:
            self._task.step_count = post
            self._task.step_count_dev = None
            act = N.Actions(h["act_dev"].data_ptr(), self.actions.data_ptr(), float(self.action_scale),
                            MODE_POSITION, 0)
            io = N.HostIO(src.data_ptr(), h["obs"].data_ptr(), h["reward"].data_ptr(), h["done"].data_ptr(),
                          h["timeout"].data_ptr(), h["poisoned"].data_ptr(), n_chunks, int(self.host_fused))
            rc = sc._sfx("bsim_env_step_host")(C.byref(lay), C.byref(par), C.byref(st), int(cfg.decimation),
                                              C.byref(act), C.byref(self._task), C.byref(io), sc._s)
            if rc != 0:
                raise N.NativeError(f"bsim_env_step_host failed ({rc}): {sc._lib.bsim_host_last_error().decode()} "
                                    f"{sc._lib.bsim_last_error().decode()}")
            h["eager_steps"] += 1
            if self.host_graph and h["eager_steps"] >= 1:   # launch configuration is warm: capture
                self._release_host_graph()
                self._task.step_count_dev = h["count_dev"].data_ptr()
                g = C.c_void_p()
                rc = sc._sfx("bsim_env_step_host_graph")(C.byref(lay), C.byref(par), C.byref(st),
                                                        int(cfg.decimation), C.byref(act), C.byref(self._task),
                                                        C.byref(io), h["count_host"].data_ptr(), C.byref(g))
                self._task.step_count_dev = None
                if rc != 0:
                    raise N.NativeError(f"bsim_env_step_host_graph failed ({rc}): "
                                        f"{sc._lib.bsim_host_last_error().decode()}")
                h["graph"], h["graph_key"] = g.value, key
        sc.step_count += cfg.decimation
        self._host_done(h, sync)
        return StepOutput(h["obs"], h["reward"], h["done"], {"timeout": h["timeout"], "poisoned": h["poisoned"]})

    def _host_done(self, h, sync):
        """Synchronise, or (sync=False) record the step so the next step_host
        waits for it before reusing the staging buffer or the graph's host
        step counter."""
        if sync:
            self.scene.stream.synchronize()
            h["inflight"] = None
            return
        ev = h.get("ev")
        if ev is None:
            ev = h["ev"] = torch.cuda.Event()
        ev.record(self.scene.stream)
        h["inflight"] = ev

    def _step_host_zero_copy(self, src, h, lay, par, st, post):
        """bsim_env_step_host mode 2: one fused launch whose CTAs read their
        actions from and write their obs / reward / flags straight to the
        pinned host buffers over PCIe (no staging copies, no chunk pipeline).
        The ctypes argument block is built once per (structs, stream); a call
        only re-points the action buffer and sets the post-step count."""
        sc = self.scene
        key = (id(lay), id(par), id(st), sc._s)
        zc = h.get("zc")
        if zc is None or zc[0] != key:
            act = N.Actions(0, self.actions.data_ptr(), float(self.action_scale), MODE_POSITION, 0)
            io = N.HostIO(0, h["obs"].data_ptr(), h["reward"].data_ptr(), h["done"].data_ptr(),
                          h["timeout"].data_ptr(), h["poisoned"].data_ptr(), 1, 2)
            args = (C.byref(lay), C.byref(par), C.byref(st), int(self.config.decimation), C.byref(act),
                    C.byref(self._task), C.byref(io), sc._s)
            zc = h["zc"] = (key, act, io, args, sc._sfx("bsim_env_step_host"))
        _, act, io, args, fn = zc
        act.actions = io.actions = src.data_ptr()
        self._task.step_count = post
        self._task.step_count_dev = None
        rc = fn(*args)
        if rc != 0:
            raise N.NativeError(f"bsim_env_step_host (zero-copy) failed ({rc}): "
                                f"{sc._lib.bsim_host_last_error().decode()} {sc._lib.bsim_last_error().decode()}")

    def _release_host_graph(self):
        h = getattr(self, "_host", None)
        if h is not None and h.get("graph"):
            self.scene._lib.bsim_host_graph_destroy(h["graph"])
            h["graph"], h["graph_key"] = None, None

    def close(self):
        self._release_host_graph()
        self.scene.close()


class QuadrupedEnv(EnvBatch):
    """Ant analog: 8-DOF walker, 60-dim obs, locomotion reward (envs.py:359-478)."""

    name = "quadruped"
    obs_dim = 60
    act_dim = 8
    action_scale = 0.6
    task_kind = TASK_QUADRUPED
    rest_height = M.QUADRUPED_REST_HEIGHT
    target_x = 1000.0

    def __init__(self, config=None):
        cfg = config or EnvConfig()
        super().__init__(replace(cfg, sim_dt=1.0 / 120.0, control_dt=1.0 / 60.0))

    def _model(self):
        return M.quadruped()

    # host-buffer step: one launch per chunk measured faster for this task
    # (16384 envs, B200: 382 vs 393 us per control step; tools/host_step_bench.py)
    host_fused = True


class AnymalObsEnv(EnvBatch):
    """ANYmal analog: 12-DOF walker, 48-dim obs, velocity tracking (envs.py:484-565)."""

    name = "quadruped-anymal-obs"
    obs_dim = 48
    act_dim = 12
    action_scale = 0.5
    task_kind = TASK_ANYMAL
    rest_height = M.QUADRUPED12_REST_HEIGHT

    def __init__(self, config=None):
        cfg = config or EnvConfig()
        super().__init__(replace(cfg, sim_dt=1.0 / 120.0, control_dt=1.0 / 60.0))

    def _model(self):
        return M.quadruped12()


class HumanoidEnv(EnvBatch):
    """Humanoid (BASELINE.json config 2): the QuadrupedEnv locomotion task
    (envs.py:359-478 obs layout, locomotion_reward, reset law) on the authored
    21-DOF capsule humanoid (models.humanoid_doc); 87-dim obs = 12 + 2x21 DOF
    + 2 foot sensors x 6 + 21 actions; done when the torso drops to 0.8 m."""

    name = "humanoid"
    obs_dim = 87
    act_dim = 21
    action_scale = 0.6
    task_kind = TASK_HUMANOID
    rest_height = M.HUMANOID_REST_HEIGHT
    termination_height = 0.8

    def __init__(self, config=None):
        cfg = config or EnvConfig()
        super().__init__(replace(cfg, sim_dt=1.0 / 120.0, control_dt=1.0 / 60.0))

    def _model(self):
        return M.humanoid()


class ShadowHandEnv(EnvBatch):
    """In-hand cube reorientation (BASELINE.json config 5, "Shadow Hand"):
    the authored 24-DOF hand (models.shadow_hand_doc: fixed forearm, coupling
    tendons, fingertip spheres, palm box) with a 6 cm cube on the palm and
    box pair contacts.  The reference has this task's reward
    (cube_reorientation_reward, rewards.py:161-176) but no env, so the env
    layer is ours: targets = 0.4 a for all 24 DOFs; 96-dim obs (layout in
    include/batchsim_b200.h, BSIM_TASK_CUBE); the cube falling 0.24 m from
    the goal point ends the episode; a success (rot_dist <= 0.4) draws a new
    goal orientation and counts in `goals[:, 7]`.  Reset: hand DOFs U(+-0.1)
    inside their limits, the cube at the spawn point with a random yaw, a
    uniform random goal orientation -- all drawn per env from PCG64 streams
    keyed (seed, global env id, reset count), like the locomotion tasks."""

    name = "shadow-hand"
    obs_dim = 2 * 24 + 24 + 24
    act_dim = 24
    action_scale = 0.4
    task_kind = TASK_CUBE

    def __init__(self, config=None):
        cfg = config or EnvConfig()
        super().__init__(replace(cfg, sim_dt=1.0 / 120.0, control_dt=1.0 / 60.0))

    def _model(self):
        return M.shadow_hand()

    def _models(self):
        return [self.model, M.cube("cube", M.SHADOW_CUBE_HALF, 0.1)]

    def _scene_kwargs(self):
        return {"shape_pairs": "all"}

    def _setup(self):
        s = self.scene
        E, B = self.config.num_envs, s.bodies_per_env
        roots = s.body_q.view(E, B, 13)
        roots[:, 0, 0:3] = torch.tensor(M.SHADOW_HAND_ROOT, dtype=s.dtype)
        self.goals[:, 0:3] = torch.tensor(M.SHADOW_CUBE_SPAWN, dtype=s.dtype)

    @property
    def successes(self):
        """Consecutive goal orientations reached in the current episode."""
        return self.goals[:, 7]


class FrankaCubeStackEnv(EnvBatch):
    """Franka cube stacking (BASELINE.json config 4): the authored 7-DOF arm
    + parallel gripper (models.franka_doc) and two free cubes (box pair
    contacts).  The reference has this task's reward (franka_stack_reward,
    rewards.py:200-219) but no env, so the env layer is ours: targets = 0.4 a
    for the 9 DOFs (the finger targets saturate at the 4 cm limit); 54-dim obs
    (layout in include/batchsim_b200.h, BSIM_TASK_STACK); a stack (cube A on
    B, aligned, gripper away) or the timeout ends the episode.  Reset: arm
    DOFs U(+-0.1) inside their limits, cube A / B at their spawn points
    + U(+-5 cm) in x and y with a random yaw, from per-env PCG64 streams
    keyed (seed, global env id, reset count)."""

    name = "franka-cube-stack"
    obs_dim = 2 * 9 + 27 + 9
    act_dim = 9
    action_scale = 0.4
    task_kind = TASK_STACK

    def __init__(self, config=None):
        cfg = config or EnvConfig()
        super().__init__(replace(cfg, sim_dt=1.0 / 120.0, control_dt=1.0 / 60.0))

    def _model(self):
        return M.franka()

    def _models(self):
        return [self.model, M.cube("cubeA", M.CUBE_A_HALF, 0.3), M.cube("cubeB", M.CUBE_B_HALF, 0.5)]

    def _scene_kwargs(self):
        return {"shape_pairs": "all"}

    def _setup(self):
        s = self.scene
        self.goals[:, 0:3] = torch.tensor(M.FRANKA_CUBE_A_SPAWN, dtype=s.dtype)
        self.goals[:, 3:6] = torch.tensor(M.FRANKA_CUBE_B_SPAWN, dtype=s.dtype)


TASKS = {
    "quadruped": QuadrupedEnv,
    "franka-cube-stack": FrankaCubeStackEnv,
    "shadow-hand": ShadowHandEnv,
    "quadruped-anymal-obs": AnymalObsEnv,
    "humanoid": HumanoidEnv,
}


def make_env(name, config=None, **overrides):
    if name not in TASKS:
        raise KeyError(f"unknown task {name!r}; have {sorted(TASKS)}")
    cfg = config or EnvConfig()
    if overrides:
        cfg = replace(cfg, **overrides)
    return TASKS[name](cfg)
