#!/bin/bash
# r02: one sweep per step-kernel instantiation (scheduled or sequential, picked by the launcher)
cd "$GRAFT_REPO_ROOT"
for i in 1 2; do
  for m in "" none; do echo "[mode ${m:-model}]"; BSIM_SCHED_MODE=$m timeout 300 python tools/quick_env_bench.py quadruped:16384 quadruped-anymal-obs:16384 humanoid:16384 shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps; done
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "step or pair or sched or sweep or envs or humanoid or shadow or franka" 2>&1 | tail -3
