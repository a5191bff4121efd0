#!/bin/bash
# r02 experiment: the joint-only schedule's in-order contact loop calls the contact rows alone
# (no second inlined copy of the joint rows in the scheduled kernels)
cd "$GRAFT_REPO_ROOT"
for v in base30 ccr base30 ccr; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py humanoid:16384 shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps; done
