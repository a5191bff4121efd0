#!/bin/bash
# r02 experiment: compile-time revolute / pass-type joint rows in the scheduled sweep (BSIM_SCHED_REV_FAST)
cd "$GRAFT_REPO_ROOT"
for v in "" revf "" revf; do
  echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py humanoid:16384 shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps
done
