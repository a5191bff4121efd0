#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in sg1 "" sg1 ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models humanoid --envs 4096,16384 --prec fp32,fp64 2>&1 | grep us/control; done
for v in sg1 ""; do BSIM_LIB_VARIANT=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1; python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads([x for x in open(f"gpurun_out/bench_{v}.log") if x.startswith("{")][-1])
oc = d.get("other_configs", {})
print(f"[{v}] " + ", ".join(f"{k} {oc[k]['value']/1e6:.2f} M" for k in ("humanoid", "franka_cube_stack", "shadow_hand", "humanoid_ppo_rollout") if k in oc))
PY
done
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_pair_shapes.py tests/test_gpu_shadow_env.py tests/test_gpu_franka_env.py tests/test_gpu_envs.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
SAN_ENVS=12 SAN_ONLY=envs,pairs timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_drive.py 2>&1 | tail -2
SAN_ENVS=12 SAN_ONLY=envs,pairs timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python tools/sanitize_drive.py 2>&1 | tail -1
