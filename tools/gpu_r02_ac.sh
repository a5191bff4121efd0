#!/bin/bash
# r02 experiment: prefetch of the next stage's row id in the scheduled sweep (BSIM_SCHED_PREFETCH)
cd "$GRAFT_REPO_ROOT"
for v in "" pf "" pf; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py humanoid:16384 humanoid:4096 2>&1 | grep env-steps; done
