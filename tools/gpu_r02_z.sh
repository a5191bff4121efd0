#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in base "" base ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12,humanoid --envs 16384 --prec fp32 2>&1 | grep us/control; BSIM_LIB_VARIANT=$v timeout 300 python tools/tail_cost.py 16384 2>&1 | grep "fused.*flush=True"; done
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -8
SAN_ENVS=20 SAN_ONLY=envs,restitution,pairs timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_drive.py 2>&1 | tail -1
