"""The model loader and the bundled robots against the reference's own.

`paper_2108_10470_b200.model.load_model` mirrors the reference loader
(/root/reference/pkg/src/batchsim/model.py:179-331: the JSON schema, the
ModelError family, DOF counts per joint kind) so a reference document loads
to the same articulation or fails with the same error class.  This runs
both loaders on the same documents -- a valid two-link arm, each joint kind,
and one mutation per validation rule -- and compares outcome for outcome;
the bundled models (models.py) are compared field by field with the
reference's factories.  CPU only; needs the reference package installed
under baseline/_ref, else skipped.
"""

import copy
import os
import sys

import numpy as np
import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "batchsim")):
        pytest.skip("reference not installed under baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import batchsim.model as RM
    import batchsim.models as RMS
    return RM, RMS


def _arm():
    return {
        "name": "arm2",
        "fixed_base": True,
        "links": [{"name": "root", "mass": 2.0, "inertia": [0.2, 0.3, 0.4]},
                  {"name": "upper", "mass": 0.7, "inertia": [0.01, 0.02, 0.02]},
                  {"name": "lower", "mass": 0.4, "inertia": [0.005, 0.01, 0.01]}],
        "joints": [{"name": "shoulder", "kind": "revolute", "parent": "root", "child": "upper", "axis": [0, 1, 0],
                    "limits": [-1.5, 1.5], "stiffness": 40.0, "damping": 2.0},
                   {"name": "elbow", "kind": "revolute", "parent": "upper", "child": "lower", "axis": [0, 1, 0]}],
        "sensors": ["lower"],
    }


def _mut(fn):
    d = copy.deepcopy(_arm())
    fn(d)
    return d


CASES = {
    "valid": _arm(),
    "prismatic": _mut(lambda d: d["joints"][1].update(kind="prismatic", axis=[1, 0, 0])),
    "spherical": _mut(lambda d: d["joints"][1].update(kind="spherical")),
    "fixed": _mut(lambda d: d["joints"][1].update(kind="fixed")),
    "zero_mass": _mut(lambda d: d["links"][2].update(mass=0.0)),
    "negative_mass": _mut(lambda d: d["links"][1].update(mass=-1.0)),
    "inverted_limits": _mut(lambda d: d["joints"][0].update(limits=[0.5, -0.5])),
    "unknown_child": _mut(lambda d: d["joints"][1].update(child="forearm")),
    "unknown_parent": _mut(lambda d: d["joints"][0].update(parent="base")),
    "loop": _mut(lambda d: d["joints"].append({"name": "back", "kind": "revolute", "parent": "lower",
                                                "child": "root", "axis": [1, 0, 0]})),
    "zero_axis": _mut(lambda d: d["joints"][0].update(axis=[0.0, 0.0, 0.0])),
    "negative_damping": _mut(lambda d: d["joints"][0].update(damping=-0.1)),
    "duplicate_link": _mut(lambda d: d["links"].append(dict(d["links"][1]))),
    "unknown_sensor": _mut(lambda d: d.update(sensors=["hand"])),
}


def _outcome(load, doc):
    try:
        m = load(copy.deepcopy(doc))
    except Exception as exc:                  # the error class is the contract
        return ("error", type(exc).__name__)
    return ("model", m.num_bodies, m.num_dofs, [j.name for j in m.joints], list(m.sensor_links))


@pytest.mark.parametrize("case", sorted(CASES))
def test_loader_matches_reference(ref, case):
    from paper_2108_10470_b200.model import load_model
    RM, _ = ref
    assert _outcome(load_model, CASES[case]) == _outcome(RM.load_model, CASES[case]), case


def test_error_family_mirrors_reference(ref):
    from paper_2108_10470_b200 import model as OM
    RM, _ = ref
    for name in ("ModelError", "CycleError", "MissingLink", "NonPositiveMass", "BadLimits"):
        ours, theirs = getattr(OM, name), getattr(RM, name)
        assert [c.__name__ for c in ours.__mro__[:-1]] == [c.__name__ for c in theirs.__mro__[:-1]], name


@pytest.mark.parametrize("name", ["free_sphere", "free_box", "flyer", "pendulum", "cartpole", "chain3",
                                  "quadruped", "quadruped12"])
def test_bundled_models_match_reference(ref, name):
    from paper_2108_10470_b200 import models as M
    _, RMS = ref
    a, b = M.get_model(name), RMS.get_model(name)
    assert (a.name, a.num_bodies, a.num_dofs, a.fixed_base) == (b.name, b.num_bodies, b.num_dofs, b.fixed_base)
    assert list(a.sensor_links) == list(b.sensor_links)
    for la, lb in zip(a.links, b.links):
        assert la.name == lb.name and np.isclose(la.mass, lb.mass) and np.allclose(la.inertia, lb.inertia)
    for ja, jb in zip(a.joints, b.joints):
        assert (ja.name, ja.kind, ja.parent, ja.child) == (jb.name, jb.kind, jb.parent, jb.child)
        assert np.allclose(ja.axis, jb.axis)
        assert (ja.limits is None) == (jb.limits is None)
        if ja.limits is not None:
            assert np.allclose(ja.limits, jb.limits)
        for f in ("stiffness", "damping", "armature", "friction"):
            assert np.isclose(getattr(ja, f), getattr(jb, f)), (name, ja.name, f)


def test_unknown_model_name_is_a_key_error(ref):
    from paper_2108_10470_b200 import models as M
    with pytest.raises(KeyError):
        M.get_model("no_such_robot")
