"""The Gauss-Seidel row schedule (SceneLayout.sweep_schedules, bsim_layout_t
.sweep_sched) keeps the reference's sequential order (physics.py:760-775):
every row of the pass appears once; rows of one stage touch disjoint bodies;
a row sharing a body with an earlier row of the reference order sits in a
later stage.  Then running a stage's rows side by side gives the sequential
values (rows on disjoint bodies commute).  The "joints" form holds the joint
rows only (the contact rows follow in order).  CPU only.
"""

import pytest

from paper_2108_10470_b200 import models as M
from paper_2108_10470_b200.layout import SceneLayout


def _scenes():
    import pair_scenes as PS
    from golden_util import build_models, load
    out = {name: SceneLayout([getattr(M, name)()], True)
           for name in ("quadruped", "quadruped12", "humanoid", "pendulum", "cartpole", "chain3")}
    out["shadow_hand_cube"] = SceneLayout([M.shadow_hand(), M.cube("cube", 0.03, 0.1)], True, "all")
    out["franka_cube_stack"] = SceneLayout(PS.SCENES["franka_cube_stack"][0](), True, "all")
    out["kitchen_sink"] = SceneLayout(build_models(load("kitchen_sink")[0]), True)
    return out


SCENES = _scenes()


def _bodies(L, r):
    J, P = L.joints_per_env, L.planes_per_env
    if r < J:
        return {L.joints[r].parent, L.joints[r].child}
    if r < J + P:
        return {int(L.plane_body[r - J])}
    a, b = L.pair_body[r - J - P]
    return {int(a), int(b)}


@pytest.mark.parametrize("mode", ["asap", "phased", "joints"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_schedule_keeps_reference_order(name, mode):
    L = SCENES[name]
    stages = L.sweep_schedules(width=4)[mode]          # a narrow width also exercises the stage splits
    n_rows = L.joints_per_env + (0 if mode == "joints" else L.planes_per_env + L.pairs_per_env)
    flat = [r for st in stages for r in st]
    assert sorted(flat) == list(range(n_rows))           # every row once
    stage_of = {r: k for k, st in enumerate(stages) for r in st}
    for st in stages:
        assert len(st) <= 4
        seen = set()
        for r in st:                                      # disjoint bodies within a stage
            b = _bodies(L, r)
            assert not (b & seen), (name, mode, st)
            seen |= b
    for r in range(n_rows):                               # dependency order = reference order
        for r2 in range(r):
            if _bodies(L, r) & _bodies(L, r2):
                assert stage_of[r2] < stage_of[r], (name, mode, r2, r)


@pytest.mark.parametrize("name", sorted(SCENES))
def test_schedule_choice(name):
    """The cost model's pick (None = the one-lane sequential sweep) matches the
    measured rankings quoted in SceneLayout.sweep_schedule."""
    L = SCENES[name]
    mode, stages, width = L.sweep_schedule()
    want = {"humanoid": "phased", "shadow_hand_cube": "joints", "franka_cube_stack": None}
    if name in want:
        assert mode == want[name], (name, mode)
    if mode is not None:
        assert stages and width == max(len(s) for s in stages)
