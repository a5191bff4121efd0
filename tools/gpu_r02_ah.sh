#!/bin/bash
# r02 experiment: scheduled contact rows out of line (BSIM_EXP_CONTACT_NOINLINE)
cd "$GRAFT_REPO_ROOT"
for v in "" cni "" cni; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py humanoid:16384 shadow-hand:16384 2>&1 | grep env-steps; done
