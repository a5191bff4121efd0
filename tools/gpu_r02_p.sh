#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for m in none asap phased joints; do
  BSIM_SCHED_MODE=$m timeout 300 python tools/quick_step_bench.py --models humanoid --envs 16384 --prec fp32 2>&1 | grep us/control | sed "s/^/[$m] /"
  BSIM_SCHED_MODE=$m timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$m.log 2>&1
  python - "$m" <<'PY'
import json, sys
m = sys.argv[1]
l = [x for x in open(f"gpurun_out/bench_{m}.log") if x.startswith("{")]
d = json.loads(l[-1]) if l else {}
oc = d.get("other_configs", {})
print(f"[{m}] " + ", ".join(f"{k} {oc[k]['value']/1e6:.2f} M" for k in ("humanoid", "franka_cube_stack", "shadow_hand") if k in oc))
PY
done
BSIM_SCHED_MODE=joints timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_pair_shapes.py tests/test_gpu_shadow_env.py tests/test_gpu_franka_env.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
