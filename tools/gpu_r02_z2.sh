#!/bin/bash
# r02 experiment: default-CTA shape for the Ant analog: 16x128 (shipped), 24x192, 32x256, 64x512
cd "$GRAFT_REPO_ROOT"
for v in "" g4 g1 g3 "" g4 g1 g3; do
  echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py quadruped:16384 quadruped:4096 quadruped:65536 2>&1 | grep env-steps
done
