#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" halves "" halves; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12 --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
BSIM_LIB_VARIANT=halves timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_envs.py tests/test_gpu_scale_parity.py tests/test_gpu_physics_kat.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
mkdir -p gpurun_out/san_halves
BSIM_LIB_VARIANT=halves SAN_ENVS=20 SAN_ONLY=envs,restitution timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_drive.py > gpurun_out/san_halves/racecheck.log 2>&1; tail -3 gpurun_out/san_halves/racecheck.log
BSIM_LIB_VARIANT=halves SAN_ENVS=20 SAN_ONLY=envs,restitution timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python tools/sanitize_drive.py > gpurun_out/san_halves/synccheck.log 2>&1; tail -2 gpurun_out/san_halves/synccheck.log
