"""Ahead-of-time topology specialisation (no JIT).

For each bundled robot the constraint topology (joint kinds, parent/child
bodies, DOF offsets, limit flags, contact-slot bodies) is emitted as a
compile-time struct into csrc/bsim_topologies.cuh; the step kernel is
instantiated once per entry so the Gauss-Seidel sweep keeps every body
velocity of an environment in registers.  Scenes whose layout matches an
entry's signature use it; anything else runs the generic kernel.

    python -m paper_2108_10470_b200.codegen     # rewrites both generated files
"""

from __future__ import annotations

import os

from . import models as M
from .layout import JOINT_KIND, SceneLayout

HERE = os.path.dirname(os.path.abspath(__file__))
CUH = os.path.join(HERE, "csrc", "bsim_topologies.cuh")
PY = os.path.join(HERE, "_topologies.py")

# name -> list of model builders (one actor each); ground plane on
SPECIALISED = {
    "quadruped": [M.quadruped],
    "quadruped12": [M.quadruped12],
}
# large articulations (the 4-env CTA of bsim_step_large.cu): the compile-time
# traits fold phase A, the sweep stays the generic shared-memory one (22+
# bodies do not fit the register-resident sweep)
SPECIALISED_LARGE = {
    "humanoid": [M.humanoid],
    # the Shadow Hand and Franka cube-stack scenes of envs.py (box / capsule
    # pair slots, shape_pairs="all"): compile-time joint kinds (the hand's
    # rows compile revolute-only), frames, tendon / pair presence, slot bodies
    "shadow_hand_cube": ([M.shadow_hand, lambda: M.cube("cube", M.SHADOW_CUBE_HALF, 0.1)], "all"),
    "franka_cube_stack": ([M.franka, lambda: M.cube("cubeA", M.CUBE_A_HALF, 0.3),
                           lambda: M.cube("cubeB", M.CUBE_B_HALF, 0.5)], "all"),
}


def signature(layout: SceneLayout):
    """Everything the specialised sweep bakes in."""
    return (layout.bodies_per_env, layout.tendons_per_env > 0, _identity_frames(layout),
            tuple((j.kind, j.parent, j.child, j.dof, int(j.has_limits)) for j in layout.joints),
            tuple(int(b) for b in layout.plane_body),
            tuple(tuple(int(x) for x in p) for p in layout.pair_body))


def _identity_frames(L):
    return all(tuple(j.origin_quat) == (0.0, 0.0, 0.0, 1.0) and tuple(j.child_quat) == (0.0, 0.0, 0.0, 1.0)
               for j in L.joints)


def _star_chain(L):
    """Chain length CH if the layout is a root with legs of CH-joint chains
    (sweep_star): joint CH l + k connects link CH l + k (root for k = 0) to
    link CH l + k + 1, all revolute with limits, dof = joint index, plane slots
    on the root then on each leg's last link, no pairs / tendons; else 0."""
    J = L.joints
    if L.pairs_per_env or L.tendons_per_env or L.bodies_per_env != len(J) + 1 or not J:
        return 0
    for ch in (2, 3):   # K lanes per env, one joint stage each (sweep_star)
        if len(J) % ch:
            continue
        ok = all(j.kind == JOINT_KIND["revolute"] and j.has_limits and j.dof == i and j.child == i + 1
                 and j.parent == (0 if i % ch == 0 else i) for i, j in enumerate(J))
        legs = len(J) // ch
        if ok and list(L.plane_body) == [0] + [ch * (l + 1) for l in range(legs)]:
            return ch
    return 0


def _arr(vals):
    vals = list(vals) or [0]
    return "{" + ", ".join(str(int(v)) for v in vals) + "}"


def _packed(vals):
    """8-bit fields, 8 per 64-bit word (entry i in byte i % 8 of word i // 8):
    the kernel unpacks entry j with a shift and a mask instead of a dependent
    load from the joint table (csrc/bsim_step.cuh unpack_u8)."""
    vals = [int(v) for v in vals] or [0]
    assert all(0 <= v < 256 for v in vals), vals
    words = []
    for w in range(0, len(vals), 8):
        x = 0
        for i, v in enumerate(vals[w:w + 8]):
            x |= v << (8 * i)
        words.append(f"{x:#x}ull")
    return "{" + ", ".join(words) + "}"


def generate():
    structs, entries, entries_large, sigs = [], [], [], []
    items = [(n, b, False) for n, b in SPECIALISED.items()] + [(n, b, True) for n, b in SPECIALISED_LARGE.items()]
    for tid, (name, spec, large) in enumerate(items, start=1):
        builders, pairs = spec if isinstance(spec, tuple) else (spec, "spheres")
        L = SceneLayout([b() for b in builders], ground=True, shape_pairs=pairs)
        J = L.joints
        cname = f"Topo_{name}"
        structs.append(f"""struct {cname} {{
    static constexpr bool is_static = true;
    static constexpr bool register_sweep = {str(not large).lower()};
    static constexpr int id = {tid};
    static constexpr int B = {L.bodies_per_env}, J = {L.joints_per_env}, P = {L.planes_per_env}, Q = {L.pairs_per_env};
    static constexpr bool all_revolute = {str(all(j.kind == JOINT_KIND["revolute"] for j in J)).lower()};
    static constexpr bool has_tendons = {str(L.tendons_per_env > 0).lower()};
    static constexpr bool identity_frames = {str(_identity_frames(L)).lower()};
    static constexpr int star_chain = {_star_chain(L)};
    static constexpr bool packed_meta = {str(L.joints_per_env <= 16).lower()};   // joint_meta from the packed tables
    static constexpr int kind[] = {_arr(j.kind for j in J)};
    static constexpr int parent[] = {_arr(j.parent for j in J)};
    static constexpr int child[] = {_arr(j.child for j in J)};
    static constexpr int dof[] = {_arr(j.dof for j in J)};
    static constexpr int limits[] = {_arr(int(j.has_limits) for j in J)};
    static constexpr int plane_body[] = {_arr(L.plane_body)};
    static constexpr int pair_a[] = {_arr(p[0] for p in L.pair_body)};
    static constexpr int pair_b[] = {_arr(p[1] for p in L.pair_body)};
    // the same tables bit-packed (8-bit entries; dof stored + 1, kl = kind | limits << 2)
    static constexpr unsigned long long parent_w[] = {_packed(j.parent for j in J)};
    static constexpr unsigned long long child_w[] = {_packed(j.child for j in J)};
    static constexpr unsigned long long dof1_w[] = {_packed(j.dof + 1 for j in J)};
    static constexpr unsigned long long kl_w[] = {_packed(j.kind | int(j.has_limits) << 2 for j in J)};
    static constexpr unsigned long long plane_body_w[] = {_packed(L.plane_body)};
}};""")
        (entries_large if large else entries).append(f"X({tid}, {cname})")
        sigs.append((tid, name, signature(L)))
    cuh = ("// GENERATED by paper_2108_10470_b200/codegen.py -- do not edit.\n"
           "// Compile-time constraint topologies of the bundled robots (see codegen.py).\n"
           "#pragma once\n\nnamespace bsim {\n\n" + "\n\n".join(structs) +
           "\n\n#define BSIM_TOPOLOGIES(X) " + " ".join(entries) +
           "\n#define BSIM_TOPOLOGIES_LARGE(X) " + " ".join(entries_large) + "\n\n}  // namespace bsim\n")
    py = ("# GENERATED by paper_2108_10470_b200/codegen.py -- do not edit.\n"
          "\"\"\"Signatures of the AOT-specialised step-kernel topologies.\"\"\"\n\n"
          "TOPOLOGIES = {\n" + "".join(f"    {sig!r}: {tid},  # {name}\n" for tid, name, sig in sigs) + "}\n")
    for path, text in ((CUH, cuh), (PY, py)):
        old = open(path).read() if os.path.exists(path) else None
        if old != text:
            with open(path, "w") as f:
                f.write(text)


def topology_id(layout: SceneLayout) -> int:
    from ._topologies import TOPOLOGIES
    return TOPOLOGIES.get(signature(layout), 0)


if __name__ == "__main__":
    generate()
    print(CUH, PY)
