#!/bin/bash
# Dev harness: for each variant (a string of extra nvcc flags, "" = baseline),
# rebuild the library on the box and time the step kernel; then parity tests.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/exp.log
: > $OUT
for v in "$@"; do
  echo "=== variant: [$v]" >> $OUT
  BSIM_NVCC_EXTRA="$v" timeout 600 python -m paper_2108_10470_b200.build --force >> $OUT 2>&1 || { echo "build failed" >> $OUT; continue; }
  timeout 300 python tools/quick_step_bench.py --envs ${QENVS:-4096,16384} --prec fp32 ${QGEN---generic} --tag "[$v] " >> $OUT 2>&1
  [ -z "$NOTEST" ] && timeout 600 python -m pytest tests/test_gpu_step.py -x -q -m gpu 2>&1 | tail -2 >> $OUT
done
cat $OUT
