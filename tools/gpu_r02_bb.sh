#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in novote "" novote ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12,humanoid --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_scale_parity.py tests/test_gpu_physics_kat.py tests/test_gpu_envs.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
