#!/bin/bash
# r02 experiment: 32-env x 256-thread default CTA as two independent 16-env groups (BSIM_SUBGROUPS=2,
# each group a full-warp sweep and its own named barrier) vs the same CTA whole and the shipped 16 x 128
cd "$GRAFT_REPO_ROOT"
for v in "" g1 g2 "" g1 g2; do
  echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py quadruped:16384 quadruped:4096 quadruped-anymal-obs:16384 2>&1 | grep env-steps
done
timeout 600 python -m pytest tests/test_gpu_ppo.py -q -p no:cacheprovider 2>&1 | tail -1
