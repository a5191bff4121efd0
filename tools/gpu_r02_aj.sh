#!/bin/bash
# r02 experiment: the joint-only schedule's contact rows chosen by a ballot over the slots' activity
cd "$GRAFT_REPO_ROOT"
for v in "" cb "" cb; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py shadow-hand:16384 humanoid:16384 2>&1 | grep env-steps; done
BSIM_LIB_VARIANT=cb timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pair or sched or shadow" 2>&1 | tail -1
