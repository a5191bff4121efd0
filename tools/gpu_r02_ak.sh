#!/bin/bash
# r02 experiment: the sequential sweep's contact rows from an activity bitmask (BSIM_SEQ_ACT_MASK)
cd "$GRAFT_REPO_ROOT"
for v in "" am "" am; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py franka-cube-stack:8192 quadruped:16384 2>&1 | grep env-steps; done
BSIM_LIB_VARIANT=am timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pair or franka or step" 2>&1 | tail -1
