#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for t in quadruped quadruped-anymal-obs; do BSIM_LIB_VARIANT=resetclk timeout 300 python tools/reset_clocks.py $t 2>&1 | tail -8; done
