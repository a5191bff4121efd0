#!/bin/bash
# r02: the sequential sweep specialised on the topology; Shadow Hand / Franka as static large topologies
cd "$GRAFT_REPO_ROOT"
for i in 1 2; do
  for m in "" none joints asap phased; do echo "[mode ${m:-model}]"; BSIM_SCHED_MODE=$m timeout 300 python tools/quick_env_bench.py shadow-hand:16384 franka-cube-stack:8192 humanoid:16384 2>&1 | grep env-steps; done
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pair or sched or shadow or franka or tendon or kitchen or step or humanoid" 2>&1 | tail -1
