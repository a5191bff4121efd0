#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" ne8m2 ne8m1 ne16m1 ne12m1 ne6m2; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models humanoid --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
for v in "" ne8m2 ne8m1 ne16m1; do BSIM_LIB_VARIANT=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1; python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/bench_{v}.log") if x.startswith("{")]
d = json.loads(l[-1]) if l else {}
oc = d.get("other_configs", {})
print(f"[{v}] " + ", ".join(f"{k} {oc[k]['value']/1e6:.2f} M" for k in ("humanoid", "franka_cube_stack", "shadow_hand", "humanoid_ppo_rollout") if k in oc))
PY
done
