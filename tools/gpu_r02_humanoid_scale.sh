#!/bin/bash
# r02: humanoid (BASELINE config 2's model) at 4096 envs -- scale parity tests + per-quantity tables (shipped + IEEE)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/hscale
timeout 1200 python -m pytest tests/test_gpu_scale_parity.py -k humanoid -q -rfE -s -p no:cacheprovider > gpurun_out/hscale/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hscale/pytest.log
grep -E "FAILED|passed|failed|rc=|ill-conditioned" gpurun_out/hscale/pytest.log | tail -8
timeout 900 python tools/parity_table.py --tasks humanoid --out gpurun_out/hscale/parity_fast.json > gpurun_out/hscale/parity_fast.log 2>&1; tail -2 gpurun_out/hscale/parity_fast.log
BSIM_LIB_VARIANT=ieee timeout 900 python tools/parity_table.py --tasks humanoid --out gpurun_out/hscale/parity_ieee.json > gpurun_out/hscale/parity_ieee.log 2>&1; tail -2 gpurun_out/hscale/parity_ieee.log
