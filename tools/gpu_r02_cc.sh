#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" d16x256 d12x192 d8x128 ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12 --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
