#!/bin/bash
# r02: double joint geometry in the fp32 step -- A/B timing (geom0 = fp32 geometry), parity (scale + drop-in), bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in geom0 "" geom0 ""; do
  BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12 --envs 4096,16384 > gpurun_out/quick_$v.log 2>&1
  echo "variant=[$v]"; cat gpurun_out/quick_$v.log | grep us/control
done
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_dropin.py -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
grep -E "PASSED|FAILED|ERROR|passed|failed|first step" gpurun_out/pytest_new.log | tail -30
timeout 900 python tools/parity_table.py --out gpurun_out/parity_fast.json > gpurun_out/parity_fast.log 2>&1; tail -2 gpurun_out/parity_fast.log
BSIM_LIB_VARIANT=ieee timeout 900 python tools/parity_table.py --out gpurun_out/parity_ieee.json > gpurun_out/parity_ieee.log 2>&1; tail -2 gpurun_out/parity_ieee.log
BSIM_LIB_VARIANT=geom0 timeout 900 python tools/parity_table.py --out gpurun_out/parity_geom0.json > gpurun_out/parity_geom0.log 2>&1; tail -2 gpurun_out/parity_geom0.log
python tools/parity_table.py --render gpurun_out/parity_fast.json gpurun_out/parity_ieee.json gpurun_out/parity_geom0.json --md gpurun_out/r02_parity_fp32.md > gpurun_out/render.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -8 gpurun_out/pytest_gpu.log
