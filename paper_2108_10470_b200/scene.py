"""GPU `Scene`: the drop-in for the reference's batched physics scene.

Same constructor, attribute names, shapes and methods as the reference
`Scene` (/root/reference/pkg/src/batchsim/physics.py:140-1091), but every
array is a torch tensor resident in HBM and every method launches a
hand-written sm_100a kernel through the C ABI (include/batchsim_b200.h).
There is no CPU fallback: constructing a Scene without CUDA or without the
built library raises.

Differences a caller can observe (all documented in DESIGN.md):

* ``pos`` / ``quat`` / ``linvel`` / ``angvel`` are views into the canonical
  env-local state ``body_q`` (position = world - env origin), which keeps
  float32 precision independent of the env grid.  ``root_state`` and
  ``body_state`` are world frame exactly as in the reference.
* ``_friction_anchor`` is stored env-local as well.
* ``step()`` is asynchronous on the scene's CUDA stream; reading a tensor
  from another stream needs ``fetch_results()`` (or torch's usual sync).
* precision="fp32" (default, fast path) or "fp64" (exact-parity path on
  B200's FP64 units).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from . import tables
from .layout import MODE_FORCE, MODE_POSITION, MODE_VELOCITY, SceneLayout
from .model import ArticulationModel
from .params import SimParams

__all__ = ["Scene", "ContactPoint", "MODE_FORCE", "MODE_POSITION", "MODE_VELOCITY"]

_STATE_TENSORS = tuple(N.STATE_PTRS)


class ContactPoint:
    """One entry of ``Scene.collide()`` (reference physics.py:95-102)."""

    __slots__ = ("body_a", "body_b", "normal", "depth", "point", "friction_anchor")

    def __init__(self, body_a, body_b, normal, depth, point, friction_anchor=None):
        self.body_a, self.body_b = int(body_a), int(body_b)
        self.normal, self.depth, self.point = normal, float(depth), point
        self.friction_anchor = friction_anchor


class Scene:
    """A batch of identical environments stepped together on one GPU."""

    def __init__(self, models, num_envs, params: SimParams | None = None, spacing=4.0,
                 ground=True, env_origins=None, device=None, precision="fp32",
                 env_offset=0, total_envs=None, stream=None, specialize=True, shape_pairs="spheres"):
        if not torch.cuda.is_available():
            raise N.NativeError("paper_2108_10470_b200.Scene needs a CUDA device (no CPU fallback)")
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(dev):       # construction launches (FK, refresh) on the scene's device
            self._init(models, num_envs, params, spacing, ground, env_origins, dev, precision, env_offset,
                       total_envs, stream, specialize, shape_pairs)

    def _init(self, models, num_envs, params, spacing, ground, env_origins, device, precision, env_offset,
              total_envs, stream, specialize, shape_pairs):
        if isinstance(models, ArticulationModel):
            models = [models]
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        self._lib = N.lib()
        self.fp64 = precision == "fp64"
        self.precision = precision
        self.dtype = torch.float64 if self.fp64 else torch.float32
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.models = list(models)
        self.num_envs = E = int(num_envs)
        self.params = (params or SimParams()).validate()
        self.ground = bool(ground)
        self.step_count = 0
        self.env_offset = int(env_offset)
        self.total_envs = int(total_envs) if total_envs is not None else self.env_offset + E

        # shape_pairs: "spheres" = the reference's contact set (sphere-sphere
        # pairs between actors); "all" adds the box / capsule pair types
        L = self.layout = SceneLayout(self.models, ground, shape_pairs)
        # AOT-specialised step kernel for known topologies (codegen.py), else generic
        from .codegen import topology_id
        self.topology_id = topology_id(L) if specialize else 0
        self.actors_per_env, self.bodies_per_env = L.actors_per_env, L.bodies_per_env
        self.dofs_per_env, self.sensors_per_env = L.dofs_per_env, L.sensors_per_env
        self.num_bodies, self.num_dofs = E * L.bodies_per_env, E * L.dofs_per_env
        self.num_actors = E * L.actors_per_env
        self.actor_body_offset = list(L.actor_body_offset)
        self.actor_dof_offset = list(L.actor_dof_offset)
        self.env_body_base = np.arange(E) * L.bodies_per_env
        self.env_dof_base = np.arange(E) * L.dofs_per_env
        self.sensor_body = L.sensor_body.copy()

        # env origins: square grid over the GLOBAL env ids (multi-GPU: same
        # origins for an env whichever rank owns it), physics.py:163-169
        if env_origins is None:
            full = L.default_env_origins(self.total_envs, spacing)
            env_origins = full[self.env_offset:self.env_offset + E]
        self.env_origins_host = np.asarray(env_origins, float).reshape(E, 3).copy()

        host = tables.init_state_arrays(L, E, self.params, self.env_origins_host, self.fp64)
        dev = self.device
        with torch.cuda.device(dev):
            self._tab = {k: torch.from_numpy(v).to(dev) for k, v in tables.pack_tables(L, self.fp64).items()}
            for k, v in host.items():
                name = "_friction_anchor" if k == "friction_anchor" else k
                object.__setattr__(self, name, torch.from_numpy(v).to(dev))
            self._env_mask = torch.zeros(max(E, 1), dtype=torch.uint8, device=dev)
            self._actor_mask = torch.zeros(1, dtype=torch.int32, device=dev)
        self._struct_cache = None
        self._struct_gen = 0
        rc = self._lib.bsim_step_smem_per_env(C.byref(self._structs()[0]), int(self.fp64), None, None)
        if rc != 0:
            raise N.NativeError(f"model too large for the step kernel (precision={precision}, rc={rc})")
        self._init_poses()

    # ------------------------------------------------------------ structs
    def __setattr__(self, name, value):
        if name in ("_struct_cache",) or not hasattr(self, "_struct_cache"):
            object.__setattr__(self, name, value)
            return
        if name in _STATE_TENSORS or name == "_friction_anchor":
            raise AttributeError(f"{name} is canonical device storage; write into it in place "
                                 f"(e.g. scene.{name}[...] = values)")
        object.__setattr__(self, name, value)

    def _structs(self):
        if self._struct_cache is None:
            ptrs = {k: v.data_ptr() for k, v in self._tab.items()}
            lay = tables.layout_struct(self.layout, self.num_envs, ptrs, self.env_offset,
                                       self.topology_id)
            sp = {}
            for name in _STATE_TENSORS:
                t = self.__dict__["_friction_anchor" if name == "friction_anchor" else name]
                sp[name] = t.data_ptr()
            st = tables.state_struct(sp)
            par = tables.params_struct(self.params, self.fp64)
            self._struct_cache = (lay, par, st)
        return self._struct_cache

    def _call(self, fn, *args, what=None):
        rc = fn(*args)
        N.check(rc, what or fn.__name__)

    def _sfx(self, name):
        return getattr(self._lib, name + ("_f64" if self.fp64 else ""))

    @property
    def _s(self):
        return self.stream.cuda_stream

    # ------------------------------------------------------------ views
    @property
    def pos(self):
        return self.body_q[:, 0:3]

    @property
    def quat(self):
        return self.body_q[:, 3:7]

    @property
    def linvel(self):
        return self.body_q[:, 7:10]

    @property
    def angvel(self):
        return self.body_q[:, 10:13]

    def set_params(self, params: SimParams):
        """Replace solver scalars (validated; takes effect on the next step)."""
        self.params = params.validate()
        self._struct_cache = None
        self._struct_gen += 1      # invalidates CUDA graphs captured with the old structs baked in

    # ------------------------------------------------------------ methods
    def _init_poses(self):
        # roots at the env origins (env-local 0), identity, then FK (physics.py:357-362)
        self.forward_kinematics()
        self.refresh_buffers()

    @N.on_scene_device
    def step(self, n_substeps: int = 1, actions=None, action_scale: float = 1.0,
             action_mode: int = MODE_POSITION, actions_clipped=None):
        """`n_substeps` x Scene.step() (physics.py:538-592) in one fused launch.

        With `actions` (E, D) device tensor: ctrl = action_scale * clip(a, -1, 1)
        is written to the position targets (or DOF forces) first -- the fused
        form of envs.py:180-187.
        """
        lay, par, st = self._structs()
        act = None
        if actions is not None:
            act = N.Actions(actions.data_ptr(), actions_clipped.data_ptr() if actions_clipped is not None else None,
                            float(action_scale), int(action_mode), 0)
        self._call(self._sfx("bsim_step"), C.byref(lay), C.byref(par), C.byref(st), int(n_substeps),
                   C.byref(act) if act is not None else None, self._s, what="bsim_step")
        self.step_count += int(n_substeps)

    @N.on_scene_device
    def forward_kinematics(self, env_mask=None, actors=None):
        """physics.py:366-425 for the selected envs / actors, plus a repack of
        the touched body/root rows."""
        lay, _, st = self._structs()
        amask = 0
        for a in range(self.actors_per_env):
            if actors is None or a in actors:
                amask |= 1 << a
        mptr = None
        if env_mask is not None:
            m = torch.as_tensor(env_mask, device=self.device).to(torch.uint8).reshape(-1)
            self._env_mask[: self.num_envs].copy_(m)
            mptr = self._env_mask.data_ptr()
        self._call(self._sfx("bsim_forward_kinematics"), C.byref(lay), C.byref(st), mptr, amask, self._s)

    @N.on_scene_device
    def refresh_buffers(self):
        """dof readout + body/root packing (physics.py:1037-1046, no contact ctx)."""
        lay, _, st = self._structs()
        self._call(self._sfx("bsim_refresh_buffers"), C.byref(lay), C.byref(st), self._s)

    @N.on_scene_device
    def read_dof_states(self):
        self.refresh_buffers()

    @N.on_scene_device
    def _set_indexed(self, root: bool, values, actor_idx):
        lay, _, st = self._structs()
        v = values.to(self.device, self.dtype).contiguous()
        idx = actor_idx.to(self.device, torch.int64).contiguous()
        fn = self._sfx("bsim_set_root_state_indexed" if root else "bsim_set_dof_state_indexed")
        self._call(fn, C.byref(lay), C.byref(st), v.data_ptr(), idx.data_ptr(), int(idx.numel()),
                   self._env_mask.data_ptr(), self._actor_mask.data_ptr(), self._s)
        return v, idx  # keep alive until the stream consumes them

    @N.on_scene_device
    def contact_geometry(self):
        """(active, depth, point, normal) per (slot, env): planes then pairs,
        env-minor, world-frame points (physics.py:463-498)."""
        lay, par, st = self._structs()
        n = (self.layout.planes_per_env + self.layout.pairs_per_env) * self.num_envs
        act = torch.zeros(max(n, 1), dtype=torch.uint8, device=self.device)
        depth = torch.zeros(max(n, 1), dtype=self.dtype, device=self.device)
        point = torch.zeros((max(n, 1), 3), dtype=self.dtype, device=self.device)
        normal = torch.zeros((max(n, 1), 3), dtype=self.dtype, device=self.device)
        self._call(self._sfx("bsim_contact_geometry"), C.byref(lay), C.byref(par), C.byref(st),
                   act.data_ptr(), depth.data_ptr(), point.data_ptr(), normal.data_ptr(), self._s)
        return act[:n].bool(), depth[:n], point[:n], normal[:n]

    @N.on_scene_device
    def collide_tensors(self, capacity=None):
        """Compacted active contacts in the reference's collide() order
        (slot-major, env-ascending, planes then pairs; physics.py:500-517) as
        device tensors: (count, body_a, body_b, depth, point, normal)."""
        lay, par, st = self._structs()
        n = (self.layout.planes_per_env + self.layout.pairs_per_env) * self.num_envs
        cap = n if capacity is None else int(capacity)
        dev = self.device
        count = torch.zeros(1, dtype=torch.int32, device=dev)
        ba = torch.zeros(max(cap, 1), dtype=torch.int32, device=dev)
        bb = torch.zeros(max(cap, 1), dtype=torch.int32, device=dev)
        depth = torch.zeros(max(cap, 1), dtype=self.dtype, device=dev)
        point = torch.zeros((max(cap, 1), 3), dtype=self.dtype, device=dev)
        normal = torch.zeros((max(cap, 1), 3), dtype=self.dtype, device=dev)
        scratch = torch.zeros(max((n + 255) // 256, 1), dtype=torch.int32, device=dev)
        self._call(self._sfx("bsim_collide"), C.byref(lay), C.byref(par), C.byref(st), cap,
                   count.data_ptr(), ba.data_ptr(), bb.data_ptr(), depth.data_ptr(), point.data_ptr(),
                   normal.data_ptr(), scratch.data_ptr(), self._s)
        k = min(int(count.item()), cap)
        return k, ba[:k], bb[:k], depth[:k], point[:k], normal[:k]

    @N.on_scene_device
    def collide(self):
        """Host list of ContactPoint in the reference's collide() order and
        content (physics.py:500-517; the friction merge of 519-534 is an
        inspection-only annotation and is applied here too)."""
        act, depth, point, normal = self.contact_geometry()
        act = act.cpu().numpy()
        depth = depth.double().cpu().numpy()
        point, normal = point.double().cpu().numpy(), normal.double().cpu().numpy()
        anchors = self._friction_anchor.double().cpu().numpy() + self.env_origins_host[None]
        L, E, B = self.layout, self.num_envs, self.bodies_per_env
        out = []
        for i in range(L.planes_per_env + L.pairs_per_env):
            for e in np.nonzero(act[i * E:(i + 1) * E])[0]:
                o = i * E + e
                if i < L.planes_per_env:
                    a = anchors[i, e]
                    out.append(ContactPoint(-1, e * B + L.plane_body[i], normal[o].copy(), depth[o],
                                            point[o].copy(), None if np.isnan(a).any() else a.copy()))
                else:
                    pa, pb = L.pair_body[i - L.planes_per_env]
                    out.append(ContactPoint(e * B + pa, e * B + pb, normal[o].copy(), depth[o],
                                            point[o].copy()))
        dmax = self.params.friction_correlation_distance
        carriers = {}
        for c in out:
            key = (c.body_a, c.body_b)
            if any(np.linalg.norm(c.point - p) < dmax for p in carriers.get(key, [])):
                c.friction_anchor = None
            else:
                carriers.setdefault(key, []).append(c.point)
        return out

    @N.on_scene_device
    def clear_nonfinite(self, env_indices):
        self.nonfinite[torch.as_tensor(env_indices, device=self.device, dtype=torch.long)] = False

    def fetch_results(self):
        """Wait for all launched work on the scene's stream (simulate/fetch split)."""
        self.stream.synchronize()

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
