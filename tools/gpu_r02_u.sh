#!/bin/bash
# r02 experiment: drive/point overlap (BSIM_DRIVE_POINT_OVERLAP) and the warp-vote limit skip
# (BSIM_LIMIT_VOTE) re-measured on the v26 kernels
cd "$GRAFT_REPO_ROOT"
for v in "" dpo lv "" dpo lv; do
  echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py quadruped:16384 quadruped-anymal-obs:16384 humanoid:16384 shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps
done
