"""DEV TOOL: where does the fp32 step's error come from?  Runs the host build
of the step kernel (tests/hostkernel, float) teacher forced from the oracle's
4096-env scale-trace pre-states (physics only, 2 substeps) against the
float64 oracle from the same states, and reports per-quantity error.  With
BSIM_HK_EXTRA set, the host build gets extra -D flags (experiments)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import scale_parity as SP  # noqa: E402


def main(task="quadruped", steps=tuple(range(20))):
    from hostkernel.hk import HostKernel
    from oracle.oracle import OracleScene
    from paper_2108_10470_b200.layout import SceneLayout
    from paper_2108_10470_b200.params import SimParams
    from oracle.tasks import OracleEnv
    meta, arr, tr = SP.oracle_trace(task)
    E = meta["num_envs"]
    env = OracleEnv(task, E, seed=0, episode_length=meta["episode_length"], threads=os.cpu_count())
    s = env.scene
    L = SceneLayout([env.model])
    hk = HostKernel(L, E, SimParams(dt=1 / 120), s.env_origins, fp64=False)
    B = s.bodies_per_env
    org = np.repeat(s.env_origins, B, axis=0)
    agg = {}
    for t in steps:
        pre = tr[t]["pre"]
        for k in ("pos", "quat", "linvel", "angvel"):
            getattr(s, k)[:] = pre[k]
        s._friction_anchor[:] = pre["anchor"]
        s.dof_state[:] = pre["dof_state"]
        tgt = (env.action_scale * np.clip(pre["actions"], -1, 1)).reshape(-1)
        s.ctrl_dof_pos_target[:] = tgt
        s.step(); s.step()
        ref = {"body": SP.local_body(s.pos, s.quat, s.linvel, s.angvel, s.env_origins, B),
               "dof_state": s.dof_state.copy(), "net_contact": s.net_contact.copy(), "dof_force": s.dof_force.copy()}
        hk.arr["body_q"][...] = SP.local_body(pre["pos"], pre["quat"], pre["linvel"], pre["angvel"], s.env_origins, B)
        hk.arr["friction_anchor"][...] = pre["anchor"] - s.env_origins[None]
        hk.arr["dof_state"][...] = pre["dof_state"]
        hk.arr["ctrl_dof_pos_target"][...] = tgt
        hk.step(2)
        got = {"body": hk.arr["body_q"].astype(float), "dof_state": hk.arr["dof_state"].astype(float),
               "net_contact": hk.arr["net_contact"].astype(float), "dof_force": hk.arr["dof_force"].astype(float)}
        for q in ref:
            e = SP.quantity_errors(got[q], ref[q], {'body': 'body_state'}.get(q, q))
            a = agg.setdefault(q, [])
            a.append(e)
            if os.environ.get("PROBE_VERBOSE"):
                print(f"  step {t:2d} {q:12s} max_abs {e['max_abs']:.2e} max_scaled {e['max_scaled']:6.2f} frac {e['frac_within']:.5f}")
    for q, es in agg.items():
        print(f"{q:12s} max_abs {max(e['max_abs'] for e in es):.3e}  p999 {max(e['p999_abs'] for e in es):.3e}  "
              f"max_scaled {max(e['max_scaled'] for e in es):6.2f}  min frac {min(e['frac_within'] for e in es):.5f}")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []))
