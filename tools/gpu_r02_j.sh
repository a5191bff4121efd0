#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" notail "" notail; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/step_overhead.py quadruped 16384 2>&1 | grep us/step; done
for ns in 1 "" ; do echo "[no_sched=$ns]"; BSIM_NO_SCHED=$ns timeout 600 python tools/quick_step_bench.py --models humanoid --envs 16384 --prec fp32 2>&1 | grep us/control; done
