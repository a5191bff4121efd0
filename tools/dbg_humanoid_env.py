"""DEV TOOL: one humanoid env of the 4096-env scale trace re-run alone on the
host build of the kernel body (fp32 and fp64) against the float64 oracle,
substep by substep: does the GPU's fp32 deviation (tools/dbg_humanoid_scale.py)
reproduce on the host, and in which substep does it appear?
    python tools/dbg_humanoid_env.py <control step> <env>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import scale_parity as SP  # noqa: E402


def main(t=10, e=1554, trace=None, restart=False):
    from hostkernel.hk import HostKernel
    from oracle.oracle import OracleScene
    from paper_2108_10470_b200 import models as M
    from paper_2108_10470_b200.layout import SceneLayout
    from paper_2108_10470_b200.params import SimParams
    meta, arr, steps = trace or SP.oracle_trace("humanoid")
    pre = steps[t]["pre"]
    model = M.humanoid()
    L = SceneLayout([model])
    B, D = L.bodies_per_env, L.dofs_per_env
    p = SimParams(dt=1.0 / 120.0)
    org = np.zeros((1, 3))
    rows = slice(e * B, (e + 1) * B)
    dr = slice(e * D, (e + 1) * D)
    E0 = meta["num_envs"]
    origins = SceneLayout([model]).default_env_origins(E0)
    pos = pre["pos"][rows] - origins[e]
    anc = pre["anchor"][:, e] - origins[e]
    tgt = 0.4 * np.clip(pre["actions"][e], -1, 1)     # action_scale (oracle/tasks.py TASK_SPECS)
    from oracle.tasks import TASK_SPECS
    tgt = TASK_SPECS["humanoid"][3] * np.clip(pre["actions"][e], -1, 1)
    o = OracleScene([model], 1, p, env_origins=org)
    o.pos[:] = pos
    o.quat[:] = pre["quat"][rows]
    o.linvel[:] = pre["linvel"][rows]
    o.angvel[:] = pre["angvel"][rows]
    o._friction_anchor[:] = anc[:, None]
    o.dof_state[:] = pre["dof_state"][dr]
    o.ctrl_dof_pos_target[:] = tgt
    hks = {}
    for name, f64 in (("hk32", False), ("hk64", True)):
        hk = HostKernel(L, 1, p, org, fp64=f64)
        hk.arr["body_q"][...] = np.concatenate([pos, pre["quat"][rows], pre["linvel"][rows], pre["angvel"][rows]], 1)
        hk.arr["friction_anchor"][...] = anc[:, None]
        hk.arr["dof_state"][...] = pre["dof_state"][dr]
        hk.arr["ctrl_dof_pos_target"][...] = tgt
        hks[name] = hk
    post = steps[t]["post"]["body_local"][rows]
    for sub in range(2):
        if restart:                                   # each substep from the oracle's exact state
            for hk in hks.values():
                if "b" in restart:
                    hk.arr["body_q"][...] = np.concatenate([o.pos, o.quat, o.linvel, o.angvel], 1)
                for ch, (c0, c1), src in (("p", (0, 3), o.pos), ("q", (3, 7), o.quat), ("l", (7, 10), o.linvel),
                                          ("w", (10, 13), o.angvel)):
                    if ch in restart:
                        hk.arr["body_q"][:, c0:c1] = src
                if "a" in restart:
                    hk.arr["friction_anchor"][...] = o._friction_anchor
                if "d" in restart:
                    hk.arr["dof_state"][...] = o.dof_state
        o.step()
        ref = np.concatenate([o.pos, o.quat, o.linvel, o.angvel], 1)
        for name, hk in hks.items():
            if os.environ.get("BSIM_DBG_MARK"):
                import ctypes
                ctypes.CDLL(None).printf(f"MARK {name} {sub}\n".encode())
            hk.step()
            g = hk.arr["body_q"].astype(float)
            d = np.abs(g - ref)
            print(f"substep {sub} {name}: max |d| {d.max():.3e} at {np.unravel_index(d.argmax(), d.shape)}; "
                  f"dof max {np.abs(hk.arr['dof_state'] - o.dof_state).max():.3e}")
    print("oracle single-env vs trace post:", np.abs(ref - post).max())
    return o, hks


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:3]], restart=sys.argv[3] if len(sys.argv) > 3 else "")
