#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for m in none asap joints; do
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
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -8
SAN_ENVS=20 SAN_ONLY=envs,pairs timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_drive.py 2>&1 | tail -1
