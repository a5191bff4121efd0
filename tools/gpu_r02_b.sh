#!/bin/bash
# r02 call B: new GPU tests (multi-rank, 4096-env parity), the parity table (fast + IEEE builds),
# racecheck per section, a bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_multirank.py -m gpu -q -rA -s > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
tail -15 gpurun_out/pytest_new.log
timeout 900 python tools/parity_table.py --out gpurun_out/parity_fast.json > gpurun_out/parity_fast.log 2>&1; tail -4 gpurun_out/parity_fast.log
BSIM_LIB_VARIANT=ieee timeout 900 python tools/parity_table.py --out gpurun_out/parity_ieee.json > gpurun_out/parity_ieee.log 2>&1; tail -4 gpurun_out/parity_ieee.log
python tools/parity_table.py --render gpurun_out/parity_fast.json gpurun_out/parity_ieee.json --md gpurun_out/r02_parity_fp32.md > /dev/null 2>&1
SAN_TOOLS=racecheck SAN_TIMEOUT=600 bash tools/gpu_sanitize.sh
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; tail -c 3000 gpurun_out/bench.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
