#!/bin/bash
# r02: Shadow Hand / Franka scenes as AOT-specialised large topologies
cd "$GRAFT_REPO_ROOT"
for i in 1 2; do
  for m in "" asap phased joints; do echo "[mode ${m:-model}]"; BSIM_SCHED_MODE=$m timeout 300 python tools/quick_env_bench.py shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps; done
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pair or sched or shadow or franka or tendon or kitchen or step" 2>&1 | tail -3
