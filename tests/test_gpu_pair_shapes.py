"""Box / capsule pair contacts on the CUDA path (shape_pairs="all"; parity
unpinned to the reference, which has none): teacher-forced steps against the
float64 C oracle's independent narrow phase, contact-query masks, and
resting-contact properties (the stacked bodies' reported contact force equals
their weight, as the reference's plane test_physics.py:208-214)."""

import numpy as np
import pytest
import torch

from golden_util import gpu_outputs, load_gpu_state, rel_err
from pair_scenes import G, SCENES, oracle_trace, setup

pytestmark = pytest.mark.gpu


def _gpu(models, p, E, precision, arr=None):
    from paper_2108_10470_b200.scene import Scene
    s = Scene(models, E, p, precision=precision, shape_pairs="all",
              env_origins=None if arr is None else arr["param_env_origins"])
    return s


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_step_matches_oracle_teacher_forced(name, precision):
    """fp64: every element within 1e-8.  fp32: every element of the root /
    body state and the contact force within 1e-3 + 1e-3 |ref| (|ref| the norm
    of the element's vector, tests/scale_parity.py) -- except elements the
    float64 reference itself cannot resolve at fp32: its output moves by at
    least 10 % of the GPU deviation when its pre-state is rounded to fp32 or
    jittered by 2^-24 relative, or when the joint-limit activations it
    decides within 8 fp32 ulps of the joint angle are re-decided at random
    (pair_scenes.oracle_sensitivity, with and without `limit_seeds`).  The
    Franka arm (light roll links in a kp-2000 drive chain, pad-cube contact
    events) and the Shadow Hand are where this matters.  The hand's fingers
    rest on their joint limits: TGS drives an engaged joint onto the limit,
    so the next passes decide the limit row at |q - limit| ~ 1e-13..1e-8
    (oracle decision margins) -- a coin flip at fp32 resolution, and a flip
    changes the finger's velocity by its whole approach rate (up to ~2 rad/s
    on gram-scale phalanges).  The reference itself, with those decisions
    re-decided, reproduces the GPU values (tools/hand_fp32_probe.py: the host
    build of the kernel, 381 + 1312 of 21216 elements excused, 0
    unexplained).  So for every scene: 0 unexplained elements; the excused
    count is 0 except on the hand, where it is reported and bounded (<= 10 %)."""
    import scale_parity as SP
    from pair_scenes import oracle_sensitivity
    models, p, meta, arr = oracle_trace(name)
    s = _gpu(models, p, meta["num_envs"], precision, arr)
    sens = oracle_sensitivity(models, p, meta, arr) if precision == "fp32" else None
    lsens = oracle_sensitivity(models, p, meta, arr, limit_seeds=tuple(range(1, 17))) if precision == "fp32" else None
    n_ill = n_bad = n_all = 0
    hand = name == "shadow_hand_cube"
    for t in range(meta["steps"]):
        load_gpu_state(s, arr, t)
        s.step()
        got = gpu_outputs(s)
        assert np.isfinite(got["body_state"]).all() and not got["nonfinite"].any(), (name, t)
        for k in ("root_state", "body_state", "net_contact"):
            if precision == "fp64":
                e = rel_err(got[k], arr[f"out_{k}"][t], 1e-8, 1e-8)
                assert e <= 1.0, (name, precision, t, k, e)
                continue
            ill, unexplained = SP.excused({k: got[k]}, {k: arr[f"out_{k}"][t]}, sens[t], k, lsens=lsens[t])
            assert unexplained == 0, (name, t, k, unexplained)
            n_ill += ill
            n_bad += unexplained
            n_all += got[k].size
    if precision == "fp32":
        print(f"{name}: {n_ill} of {n_all} elements beyond 1e-3 and ill-conditioned in the reference itself, "
              f"{n_bad} beyond 1e-3 otherwise")
        if hand:
            # fingers on their limits (docstring): excused elements reported and bounded
            assert n_ill <= 0.10 * n_all, (n_ill, n_all)
        else:
            assert n_ill == 0, (name, n_ill)


@pytest.mark.parametrize("name", sorted(SCENES))
def test_contact_geometry_masks_match_oracle(name):
    """Active masks of every plane / pair slot are identical to the oracle's
    (depths / points / normals within fp64 rounding)."""
    from oracle.oracle import OracleScene
    models, p, meta, arr = oracle_trace(name, steps=2)
    ref = OracleScene(models, meta["num_envs"], p, shape_pairs="all", env_origins=arr["param_env_origins"])
    for k in ("pos", "quat", "linvel", "angvel"):
        getattr(ref, k)[...] = arr[f"out_{k}"][-1]
    s = _gpu(models, p, meta["num_envs"], "fp64", arr)
    load_gpu_state(s, arr, 1, prefix="out_")
    ga, gd, gp, gn = (x.cpu().numpy() if isinstance(x, torch.Tensor) else x for x in s.contact_geometry())
    ra, rd, rp, rn = ref.contact_geometry()
    assert np.array_equal(np.asarray(ga, bool), np.asarray(ra, bool))
    np.testing.assert_allclose(gd, rd, atol=1e-9)
    np.testing.assert_allclose(gp, rp, atol=1e-9)
    np.testing.assert_allclose(gn, rn, atol=1e-9)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", sorted(n for n in SCENES if n not in ("franka_cube_stack", "shadow_hand_cube")))
def test_resting_pair_contact_carries_weight(name, precision):
    """After settling, each body's reported net contact force, averaged over
    1 s, equals its own weight (the lower body's ground force minus the load
    on top), and the stack holds its height."""
    from paper_2108_10470_b200.params import SimParams
    models = SCENES[name][0]()
    E = 4
    s = _gpu(models, SimParams(dt=1 / 120), E, precision)
    setup(name, s)
    z0 = s.pos[:, 2].double().clone()
    s.step(240)
    B = s.bodies_per_env
    acc = torch.zeros(E * B, dtype=torch.float64, device=s.device)
    for _ in range(120):
        s.step()
        acc += s.net_contact[:, 2].double()
    w = torch.as_tensor(np.tile([sum(l.mass for l in m.links) * G for m in models], E), device=s.device)
    dyn = s.inv_mass > 0                       # static rails carry no weight of their own
    assert float(((acc / 120 - w).abs() / w)[dyn].max()) < 0.05, (acc / 120 / w)
    assert float((s.pos[:, 2].double() - z0).abs().max()) < 0.01


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_franka_cubes_rest_under_held_arm(precision):
    """Franka cube-stack scene: with the arm PD-held at its home pose (pads
    above the cubes) both cubes rest on the ground -- their reported contact
    force is their weight -- and the gripper pads stay clear of them."""
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.params import SimParams
    models = SCENES["franka_cube_stack"][0]()
    E = 8
    s = _gpu(models, SimParams(dt=1 / 120), E, precision)
    setup("franka_cube_stack", s)
    s.step(240)
    B = s.bodies_per_env
    acc = torch.zeros((E, 2), dtype=torch.float64, device=s.device)
    for _ in range(120):
        s.step()
        acc += s.net_contact[:, 2].double().reshape(E, B)[:, 10:12]
    w = torch.tensor([0.3 * G, 0.5 * G], dtype=torch.float64, device=s.device)
    assert float(((acc / 120 - w).abs() / w).max()) < 0.03
    assert bool(torch.isfinite(s.body_q).all()) and int(s.nonfinite.sum()) == 0


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_shadow_hand_holds_cube_on_palm(precision):
    """Shadow Hand scene at rest (PD holding the open hand): the cube rests on
    the palm -- its contact force is its weight, it stays above the palm."""
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.params import SimParams
    models = SCENES["shadow_hand_cube"][0]()
    E = 8
    s = _gpu(models, SimParams(dt=1 / 120), E, precision)
    setup("shadow_hand_cube", s)
    s.step(120)
    B = s.bodies_per_env
    acc = torch.zeros(E, dtype=torch.float64, device=s.device)
    for _ in range(60):
        s.step()
        acc += s.net_contact[:, 2].double().reshape(E, B)[:, B - 1]
    w = 0.1 * G
    assert float(((acc / 60 - w).abs() / w).max()) < 0.05
    z = s.pos[:, 2].double().reshape(E, B)[:, B - 1]
    assert float(z.min()) > M.SHADOW_HAND_ROOT[2]
