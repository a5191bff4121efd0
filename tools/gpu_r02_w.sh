#!/bin/bash
# r02 experiment: code-size probe -- the scheduled sweep compiled out (BSIM_EXP_NO_SCHED_CODE); Franka
# runs the sequential sweep either way
cd "$GRAFT_REPO_ROOT"
for v in "" nosched "" nosched; do
  echo "[$v]"; BSIM_SCHED_MODE=none BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py humanoid:16384 shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps
done
