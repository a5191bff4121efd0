"""Flatten a list of actor models into the per-env tables the kernels consume.

Host-side, built once per scene.  Index conventions follow the reference
`Scene` layout (`pkg/src/batchsim/physics.py:216-355`):

* bodies of one env are contiguous, actor after actor; global body row
  ``e * B + actor_body_offset[a] + link`` (physics.py:229-230, 271-272);
* DOFs likewise, ``e * D + actor_dof_offset[a] + dof`` (physics.py:282);
* joint slots are ordered actor-major, then depth-first joint order
  (physics.py:262-287); each pass solves all joints, then plane slots, then
  pair slots (physics.py:761-775);
* collision slots: sphere -> 1 plane slot, capsule -> 2 end spheres, box -> 8
  corner points with radius 0 (physics.py:314-327); sphere-sphere pair slots
  between different actors of the same env (physics.py:331-338);
* a fixed-base root link has inv_mass 0 and zero inertia (physics.py:236-238);
* a DOF is in POSITION mode iff its joint stiffness > 0 (physics.py:288-289).

Every table is a plain numpy array; ``joint_table()`` packs the joint rows in
the C struct layout ``bsim_joint_t`` declared in ``include/batchsim_b200.h``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import ArticulationModel

JOINT_KIND = {"fixed": 0, "revolute": 1, "prismatic": 2, "spherical": 3}
MODE_FORCE, MODE_POSITION, MODE_VELOCITY = 0, 1, 2
MODES = {"force": MODE_FORCE, "position": MODE_POSITION, "velocity": MODE_VELOCITY}

# bsim_joint_t: 8 int32 then 24 float32 (128 bytes)
JOINT_INTS = 8
JOINT_FLOATS = 24
# bsim_tendon_t / bsim_tendon_elem_t sizes (see header)
TENDON_INTS = 8
TENDON_FLOATS = 8
TELEM_INTS = 4
TELEM_FLOATS = 4


@dataclass
class JointRow:
    kind: int
    parent: int        # local body index within the env
    child: int
    dof: int           # local DOF offset within the env, -1 for fixed joints
    actor: int
    has_limits: bool
    axis: np.ndarray
    origin_pos: np.ndarray
    origin_quat: np.ndarray
    child_pos: np.ndarray
    child_quat: np.ndarray
    stiffness: float
    damping: float
    armature: float
    friction: float
    limit_lo: float
    limit_hi: float


PAIR_SS, PAIR_PB, PAIR_PC, PAIR_CC = 0, 1, 2, 3      # bsim_pair_kind (include/batchsim_b200.h)


def _corners(sh):
    hx, hy, hz = sh.params
    off = np.asarray(sh.offset, float)
    return [off + [sx * hx, sy * hy, sz * hz] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]


def _ends(sh):
    r, hh = sh.params
    off = np.asarray(sh.offset, float)
    return [off + [0.0, 0.0, s * hh] for s in (-1.0, 1.0)]


def pair_slots(b1, s1, b2, s2):
    """Candidate contact slots of one shape pair between two actors:
    (kind, body_a, off_a, rad_a, body_b, off_b, rad_b, ext4).

    sphere-sphere is the reference's pair (physics.py:330-338, one SS slot,
    a = the first shape).  The box / capsule pairs extend the same static-slot
    model the reference uses for the ground (physics.py:314-327: capsule ->
    two end spheres, box -> eight corner points): sphere-box one PB slot;
    capsule-box the capsule's end spheres against the box (2 PB) and the box
    corners against the capsule (8 PC); box-box each box's corners against
    the other box (16 PB); sphere-capsule one PC slot; capsule-capsule one CC
    slot (segment-segment)."""
    z4 = (0.0, 0.0, 0.0, 0.0)
    off = lambda sh: np.asarray(sh.offset, float)  # noqa: E731

    def pb(ba, pa_, ra_, bb, sb):          # point/sphere on ba vs box sb on bb
        return (PAIR_PB, ba, pa_, ra_, bb, off(sb), 0.0, (*sb.params, 0.0))

    def pc(ba, pa_, ra_, bb, sb):          # point/sphere on ba vs capsule sb on bb
        return (PAIR_PC, ba, pa_, ra_, bb, off(sb), sb.params[0], (0.0, sb.params[1], 0.0, 0.0))

    k1, k2 = s1.kind, s2.kind
    if k1 == "sphere" and k2 == "sphere":
        return [(PAIR_SS, b1, off(s1), s1.params[0], b2, off(s2), s2.params[0], z4)]
    if k1 == "box" and k2 != "box":        # order so that a box, if any, is the second shape
        return pair_slots(b2, s2, b1, s1)
    if k1 == "capsule" and k2 == "sphere":
        return pair_slots(b2, s2, b1, s1)
    if k1 == "sphere" and k2 == "box":
        return [pb(b1, off(s1), s1.params[0], b2, s2)]
    if k1 == "sphere" and k2 == "capsule":
        return [pc(b1, off(s1), s1.params[0], b2, s2)]
    if k1 == "capsule" and k2 == "capsule":
        return [(PAIR_CC, b1, off(s1), s1.params[0], b2, off(s2), s2.params[0], (s1.params[1], s2.params[1], 0.0, 0.0))]
    if k1 == "capsule" and k2 == "box":
        return ([pb(b1, e, s1.params[0], b2, s2) for e in _ends(s1)] +
                [pc(b2, c, 0.0, b1, s1) for c in _corners(s2)])
    if k1 == "box" and k2 == "box":
        return ([pb(b1, c, 0.0, b2, s2) for c in _corners(s1)] +
                [pb(b2, c, 0.0, b1, s1) for c in _corners(s2)])
    return []


class SceneLayout:
    """Per-env tables for a list of actors replicated over all envs."""

    def __init__(self, models, ground=True, shape_pairs="spheres"):
        if isinstance(models, ArticulationModel):
            models = [models]
        self.models = list(models)
        self.ground = bool(ground)
        self.actors_per_env = len(self.models)
        self.actor_body_offset, self.actor_dof_offset = [], []
        b = d = 0
        for m in self.models:
            self.actor_body_offset.append(b)
            self.actor_dof_offset.append(d)
            b += m.num_bodies
            d += m.num_dofs
        self.bodies_per_env, self.dofs_per_env = b, d

        # bodies
        B = self.bodies_per_env
        self.body_actor = np.zeros(B, np.int32)
        self.inv_mass = np.zeros(B)
        self.inertia = np.zeros((B, 3))
        for a, m in enumerate(self.models):
            for li, link in enumerate(m.links):
                gi = self.actor_body_offset[a] + li
                self.body_actor[gi] = a
                if not (m.fixed_base and li == 0):
                    self.inv_mass[gi] = 1.0 / link.mass
                    self.inertia[gi] = link.inertia
        pos = self.inertia > 0
        self.inv_inertia = np.where(pos, 1.0 / np.where(pos, self.inertia, 1.0), 0.0)

        # joints
        self.joints: list[JointRow] = []
        self.dof_mode = np.zeros(self.dofs_per_env, np.int8)
        self.dof_joint = np.zeros(self.dofs_per_env, np.int32)
        self.dof_lower = np.full(self.dofs_per_env, -np.inf)
        self.dof_upper = np.full(self.dofs_per_env, np.inf)
        for a, m in enumerate(self.models):
            boff, doff = self.actor_body_offset[a], self.actor_dof_offset[a]
            cursor = 0
            for j in m.joints:
                dof = -1
                if j.dof_count:
                    dof = doff + cursor
                    for k in range(j.dof_count):
                        self.dof_joint[dof + k] = len(self.joints)
                        if j.limits:
                            self.dof_lower[dof + k], self.dof_upper[dof + k] = j.limits
                    cursor += j.dof_count
                    if j.stiffness > 0:
                        self.dof_mode[dof] = MODE_POSITION
                lo, hi = j.limits if j.limits else (-np.inf, np.inf)
                self.joints.append(JointRow(
                    JOINT_KIND[j.kind], boff + m.link_index(j.parent), boff + m.link_index(j.child),
                    dof, a, j.limits is not None, np.asarray(j.axis, float),
                    np.asarray(j.origin_pos, float), np.asarray(j.origin_quat, float),
                    np.asarray(j.child_pos, float), np.asarray(j.child_quat, float),
                    j.stiffness, j.damping, j.armature, j.friction, lo, hi))
        self.joints_per_env = len(self.joints)

        # collision slots
        shapes = []
        for a, m in enumerate(self.models):
            for li, link in enumerate(m.links):
                if link.shape is not None and link.collision and link.shape.kind != "none":
                    shapes.append((a, self.actor_body_offset[a] + li, link.shape))
        plane = []
        for _, body, sh in shapes:
            off = np.asarray(sh.offset, float)
            if sh.kind == "sphere":
                plane.append((body, off, sh.params[0]))
            elif sh.kind == "capsule":
                r, hh = sh.params
                plane += [(body, off + [0.0, 0.0, s * hh], r) for s in (-1.0, 1.0)]
            elif sh.kind == "box":
                hx, hy, hz = sh.params
                plane += [(body, off + [sx * hx, sy * hy, sz * hz], 0.0)
                          for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]
        if not self.ground:
            plane = []
        self.plane_body = np.array([p[0] for p in plane], np.int32)
        self.plane_off = np.array([p[1] for p in plane], float).reshape(-1, 3)
        self.plane_rad = np.array([p[2] for p in plane], float)
        pairs = []
        for i in range(len(shapes)):
            for k in range(i + 1, len(shapes)):
                (ai, bi, si), (ak, bk, sk) = shapes[i], shapes[k]
                if ai == ak:          # self-collision within an actor is off (physics.py:333-334)
                    continue
                if shape_pairs == "spheres":   # the reference's pair set (physics.py:335-338)
                    if si.kind == "sphere" and sk.kind == "sphere":
                        pairs += pair_slots(bi, si, bk, sk)
                elif shape_pairs == "all":     # + box / capsule pair types (extension)
                    pairs += pair_slots(bi, si, bk, sk)
                else:
                    raise ValueError("shape_pairs must be 'spheres' (reference) or 'all'")
        self.pair_kind = np.array([p[0] for p in pairs], np.int32)
        self.pair_body = np.array([[p[1], p[4]] for p in pairs], np.int32).reshape(-1, 2)
        self.pair_off = np.array([[p[2], p[5]] for p in pairs], float).reshape(-1, 2, 3)
        self.pair_rad = np.array([[p[3], p[6]] for p in pairs], float).reshape(-1, 2)
        self.pair_ext = np.array([p[7] for p in pairs], float).reshape(-1, 4)
        self.planes_per_env = len(plane)
        self.pairs_per_env = len(pairs)

        # sensors
        sens = []
        for a, m in enumerate(self.models):
            for name in (m.sensor_links or ()):
                sens.append(self.actor_body_offset[a] + m.link_index(name))
        self.sensor_body = np.array(sens, np.int32)
        self.sensors_per_env = len(sens)

        self._build_tendons()

    # ------------------------------------------------------------ tendons
    def _build_tendons(self):
        """Fixed tendons (reference tendons.py:65-95, physics.py:598-653) and
        spatial tendons (tendons.py:148-188) flattened into rows + elements."""
        rows, elems = [], []
        for a, m in enumerate(self.models):
            boff, doff = self.actor_body_offset[a], self.actor_dof_offset[a]
            dof_of = {}
            c = 0
            for j in m.joints:
                if j.dof_count:
                    dof_of[j.name] = c
                    c += j.dof_count
            for spec in m.tendons:
                lo, hi = spec.limits if spec.limits else (0.0, 0.0)
                first = len(elems)
                if spec.kind == "fixed":
                    root_joint = m.joints[m.joint_index(spec.joints[0].dof)]
                    reaction = boff + m.link_index(root_joint.parent)
                    for tj in spec.joints:
                        ji = m.joint_index(tj.dof)
                        joint_slot = self._joint_slot(a, ji)
                        elems.append(((doff + dof_of[tj.dof], tj.parent, joint_slot, 0),
                                      (tj.coefficient, 0.0, 0.0, 0.0)))
                    kind = 0
                else:
                    for at in spec.attachments:
                        elems.append(((boff + m.link_index(at.link), at.parent, 0, 0),
                                      (at.offset[0], at.offset[1], at.offset[2], at.weight)))
                    reaction = -1
                    kind = 1
                rows.append(((kind, first, len(elems) - first, int(spec.limits is not None),
                              reaction, a, 0, 0),
                             (spec.rest_length, spec.stiffness, spec.damping, lo, hi,
                              spec.limit_stiffness, 0.0, 0.0)))
        self.tendons_per_env = len(rows)
        self.tendon_int = np.array([r[0] for r in rows], np.int32).reshape(-1, TENDON_INTS)
        self.tendon_flt = np.array([r[1] for r in rows], np.float64).reshape(-1, TENDON_FLOATS)
        self.telem_int = np.array([e[0] for e in elems], np.int32).reshape(-1, TELEM_INTS)
        self.telem_flt = np.array([e[1] for e in elems], np.float64).reshape(-1, TELEM_FLOATS)
        # spatial sub-tendon paths (root-to-leaf, declaration order), as element indices
        self.spatial_paths = []
        for t in range(self.tendons_per_env):
            kind, first, count = self.tendon_int[t, :3]
            if kind != 1:
                self.spatial_paths.append([])
                continue
            parents = [int(self.telem_int[first + i, 1]) for i in range(count)]
            kids = {i: [k for k in range(count) if parents[k] == i] for i in range(count)}
            root = parents.index(-1)
            paths = []

            def walk(i, path):
                path = path + [i]
                if not kids[i]:
                    paths.append(path)
                for k in kids[i]:
                    walk(k, path)
            walk(root, [])
            self.spatial_paths.append(paths)

    def _joint_slot(self, actor, joint_index):
        n = 0
        for a in range(actor):
            n += len(self.models[a].joints)
        return n + joint_index

    # ------------------------------------------------------------ packing
    def _sched_rows(self):
        J, P = self.joints_per_env, self.planes_per_env
        rows = [(j, {jt.parent, jt.child}) for j, jt in enumerate(self.joints)]
        rows += [(J + i, {int(b)}) for i, b in enumerate(self.plane_body)]
        rows += [(J + P + q, {int(a), int(b)}) for q, (a, b) in enumerate(self.pair_body)]
        return rows

    def _levels(self, rows, phased, width):
        """ASAP stages of `rows` (reference order): row r goes to 1 + the
        stage of the last earlier row sharing a body with it; `phased`: no
        contact row before the last joint stage."""
        J = self.joints_per_env
        last, stage_of, floor = {}, [], 0
        for r, bodies in rows:
            if phased and r == J:
                floor = max(stage_of, default=-1) + 1
            st = max(floor, 1 + max(last.get(b, -1) for b in bodies))
            stage_of.append(st)
            for b in bodies:
                last[b] = st
        out = []
        for k in range(max(stage_of) + 1 if stage_of else 0):
            st = [r for (r, _), s in zip(rows, stage_of) if s == k]
            out += [st[i:i + width] for i in range(0, len(st), width)]
        return out

    def sweep_schedules(self, width=32):
        """The candidate row schedules of one Gauss-Seidel pass
        (physics.py:760-775: joints, then plane slots, then pair slots, each in
        index order).  Rows of a stage touch disjoint bodies and every row runs
        after each earlier row it shares a body with, so running a stage's
        rows side by side (one lane each) reproduces the sequential sweep
        exactly (rows on disjoint bodies commute).  Row ids: joint j -> j,
        plane slot i -> J + i, pair slot q -> J + P + q.
          "asap":   all rows, ASAP stages;
          "phased": all rows, contact rows only after the last joint stage
                    (stages of one row type: no divergence in a warp);
          "joints": the joint rows only (sched_flags bit 0: the contact rows
                    follow in reference order on one lane -- every contact
                    row comes after every joint row in the reference order).
        Stages wider than `width` are split."""
        rows = self._sched_rows()
        J = self.joints_per_env
        return {"asap": self._levels(rows, False, width), "phased": self._levels(rows, True, width),
                "joints": self._levels(rows[:J], False, width)}

    def _sched_cost(self, mode, stages, lanes=2, per_stage=0.3, contact=0.5, mixed=0.5):
        """Modelled row times of a pass: per stage, the costliest row type
        present (joint / plane / pair) costs ceil(rows of the type / lanes),
        each further type `mixed` x its own (divergent paths of a warp partly
        overlap), plus `per_stage` (schedule load, __syncwarp); a contact row
        counts `contact` (inactive slots skip, BSIM_SKIP_INACTIVE); mode
        "joints" adds its sequential contact rows.  The weights are fitted to
        the measured mode rankings quoted in sweep_schedule."""
        J, P, Q = self.joints_per_env, self.planes_per_env, self.pairs_per_env
        cost = 0.0
        for st in stages:
            n = [0, 0, 0]
            for r in st:
                n[0 if r < J else (1 if r < J + P else 2)] += 1
            ts = sorted((-(-k // lanes) * (1.0 if t == 0 else contact) for t, k in enumerate(n) if k), reverse=True)
            cost += per_stage + (ts[0] + mixed * sum(ts[1:]) if ts else 0.0)
        if mode == "joints":
            cost += contact * (P + Q)
        return cost

    def _sweep_lanes(self):
        """Lanes per env the kernel gives the schedule: 16 on the large-
        articulation CTA (8 envs on 4 sweep warps, BSIM_LARGE_SCHED_WARPS), 2
        on the default one (16 envs share one warp).  Mirrors csrc: make_dims' record size (BODY 36, JOINT 44,
        PLANE 28, PAIR 76, ANCHOR 4, DOF 2 items, ENV 8, pad = 4 mod 8) and
        use_large_variant (a 16-env fp32 workspace over 113 KB)."""
        items = (36 * self.bodies_per_env + 44 * self.joints_per_env + 28 * self.planes_per_env +
                 76 * self.pairs_per_env + 4 * self.planes_per_env + 2 * self.dofs_per_env)
        items = ((items + 3) & ~3) + 8
        while items % 8 != 4:
            items += 1
        return 16 if 16 * items * 4 > 113 * 1024 else 2

    def sweep_schedule(self, width=32):
        """(mode, stages, width) of the schedule the kernel runs, or mode
        None: the sequential one-lane sweep.  The cheapest candidate by the
        cost model (on the kernel's lanes per env, _sweep_lanes), used when it
        is below 0.8 of the sequential cost.  Measured on B200, fp32, every
        mode forced, on the v29 kernels (16 lanes per env on the large CTA,
        one sweep per kernel instantiation, rows specialised on the
        compile-time topology; tools/gpu_r02_ae.sh): humanoid 16384 envs
        none / asap / phased / joints 1482 / 1397 / 1340 / 1537 us per
        control step -> phased; Shadow Hand 4.78 / 4.13 / 3.97 / 5.03 M
        env-steps/s -> joints; Franka cube-stack 9.35 / 6.90 / 6.50 / 7.07 M
        -> none.  The model picks the same three (the hand's joints form
        models at 0.78 of its sequential cost; with round 2's earlier kernels
        it measured slower than the sequential sweep and 0.75 was used:
        tools/gpu_r02_x.sh; with 4 lanes per env the humanoid picked asap:
        tools/gpu_r02_p.sh).
        BSIM_SCHED_MODE=asap|phased|joints|none forces a mode (experiments,
        tests/test_gpu_sched_modes.py); read once per layout: the result is
        memoised, so the packed table and the layout struct always agree."""
        import os
        memo = self.__dict__.setdefault("_sched_memo", {})
        if width not in memo:
            memo[width] = self._pick_schedule(width, os.environ.get("BSIM_SCHED_MODE"))
        return memo[width]

    def _pick_schedule(self, width, forced):
        cands = self.sweep_schedules(width)
        J = self.joints_per_env
        seq = J + 0.5 * (self.planes_per_env + self.pairs_per_env)
        if forced:
            mode = None if forced == "none" else forced
        else:
            lanes = self._sweep_lanes()
            mode = min(cands, key=lambda m: self._sched_cost(m, cands[m], lanes))
            if not cands[mode] or self._sched_cost(mode, cands[mode], lanes) >= 0.8 * seq:
                mode = None
        if mode is None:
            return None, [], 0
        st = cands[mode]
        return mode, st, max((len(s) for s in st), default=0)

    def joint_table(self):
        """(J, 8) int32 and (J, 24) float32 views of bsim_joint_t rows."""
        J = self.joints_per_env
        ints = np.zeros((J, JOINT_INTS), np.int32)
        flts = np.zeros((J, JOINT_FLOATS), np.float64)
        for i, j in enumerate(self.joints):
            ints[i, :6] = (j.kind, j.parent, j.child, j.dof, j.actor, int(j.has_limits))
            flts[i, 0:3] = j.axis
            flts[i, 3:6] = j.origin_pos
            flts[i, 6:10] = j.origin_quat
            flts[i, 10:13] = j.child_pos
            flts[i, 13:17] = j.child_quat
        return ints, flts

    def joint_param_defaults(self):
        """(6, J): stiffness, damping, armature, friction, limit_lo, limit_hi."""
        return np.array([[j.stiffness for j in self.joints], [j.damping for j in self.joints],
                         [j.armature for j in self.joints], [j.friction for j in self.joints],
                         [j.limit_lo for j in self.joints], [j.limit_hi for j in self.joints]],
                        float).reshape(6, self.joints_per_env)

    def default_env_origins(self, num_envs, spacing=4.0):
        """Square grid, cols = ceil(sqrt(E)) (physics.py:163-169)."""
        cols = int(np.ceil(np.sqrt(num_envs)))
        e = np.arange(num_envs)
        return np.stack([spacing * (e % cols), spacing * (e // cols), np.zeros(num_envs)], -1)
