#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in nodpo "" nodpo ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12,humanoid --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -8
timeout 900 python tools/parity_table.py --out gpurun_out/parity_dpo.json > gpurun_out/parity_dpo.log 2>&1; tail -1 gpurun_out/parity_dpo.log
