#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for i in 1 2; do BSIM_LIB_VARIANT=phaseclk timeout 300 python tools/launch_gap.py quadruped 16384 2>&1 | tail -2; done
BSIM_LIB_VARIANT=phaseclk timeout 300 python tools/step_overhead.py quadruped 16384 2>&1 | grep us/step
BSIM_LIB_VARIANT=phaseclk timeout 300 python tools/cta_timeline.py quadruped 16384 2>&1 | grep -E "span"
