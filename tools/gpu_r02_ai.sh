#!/bin/bash
# r02 experiment: joint kinds folded onto the kinds the compile-time topology contains (fold_kind)
cd "$GRAFT_REPO_ROOT"
for v in "" fk "" fk; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py franka-cube-stack:8192 humanoid:16384 shadow-hand:16384 quadruped:16384 2>&1 | grep env-steps; done
