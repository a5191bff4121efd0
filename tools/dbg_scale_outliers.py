"""DEV TOOL: where a task's fp32 elements beyond 1e-3 sit at 4096 envs
(teacher forced vs the float64 oracle): per step the envs, bodies / DOFs and
columns, the GPU deviation, the reference's own spread under fp32-sized
input noise with 2 seeds and with N seeds plus N knife-edge limit
re-decisions, and whether the env reset.
    python tools/dbg_humanoid_scale.py <task> <out.json>"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import scale_parity as SP  # noqa: E402


def main(task="humanoid", nseeds=16, out=None):
    trace = SP.oracle_trace(task)
    meta, arr, steps = trace
    _, _, res = SP.teacher_forced(task, "fp32", trace)
    s2 = SP.sensitivity(task, trace)
    sN = SP.sensitivity(task, trace, seeds=tuple(range(1, nseeds + 1)))
    lN = SP.limit_sensitivity(task, trace, seeds=tuple(range(1, nseeds + 1)))
    sN = [{q: np.maximum(a[q], b[q]) for q in a} for a, b in zip(sN, lN)]
    B, D, S = SP.sample_dims(arr)
    per = {"body_state": B, "root_state": 1, "dof_state": D, "dof_force": D, "net_contact": B, "sensor_forces": S, "obs": 1,
           "reward": 1}
    rows = []
    tot2 = totN = 0
    for t, r in enumerate(res):
        done = r["ref"]["done"]
        for q in SP.QUANTITIES:
            _, u2 = SP.excused(r["gpu"], r["ref"], s2[t], q)
            _, uN = SP.excused(r["gpu"], r["ref"], sN[t], q)
            tot2 += u2
            totN += uN
            if not uN:
                continue
            g = np.asarray(r["gpu"][q], float)
            f = np.asarray(r["ref"][q], float)
            f2 = f.reshape(len(f), -1)
            g2 = g.reshape(f2.shape)
            d = np.abs(g2 - f2)
            sc = d / (SP.ATOL + SP.RTOL * SP._magnitude(q, f2))
            sn = np.asarray(sN[t][q], float).reshape(f2.shape)
            bad = np.argwhere((sc > 10) & (sn < 0.1 * d))
            k = per.get(q, 1)
            envs = sorted({int(i // k) for i, _ in bad})
            rows.append({"t": t, "q": q, "unexplained_2": u2, "unexplained_N": uN, "envs": envs[:20],
                         "n_envs": len(envs), "env_done": [bool(done[e]) for e in envs[:20]],
                         "worst": [{"row": int(i), "col": int(c), "gpu": float(g2[i, c]), "ref": float(f2[i, c]),
                                    "d": float(d[i, c]), "sensN": float(sn[i, c])}
                                   for i, c in bad[np.argsort(-d[bad[:, 0], bad[:, 1]])][:5]]})
            print(json.dumps(rows[-1]), flush=True)
    print(f"unexplained with 2 seeds {tot2}, with {nseeds} seeds {totN}")
    if out:
        json.dump(rows, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "humanoid", out=sys.argv[2] if len(sys.argv) > 2 else None)
