#!/bin/bash
# r02 experiment: the row-schedule sweep on 1 / 2 / 4 warps of the large CTA (BSIM_LARGE_SCHED_WARPS:
# 4 / 8 / 16 lanes per env), every schedule mode forced
cd "$GRAFT_REPO_ROOT"
for v in "" sw2 sw4; do
  for m in asap phased joints none; do
    echo "[$v $m]"; BSIM_SCHED_MODE=$m BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py humanoid:16384 shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps
  done
done
