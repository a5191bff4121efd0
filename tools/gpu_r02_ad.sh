#!/bin/bash
# r02: scheduled sweep rows specialised on the compile-time topology (humanoid: revolute rows only, no pair rows)
cd "$GRAFT_REPO_ROOT"
for i in 1 2; do timeout 300 python tools/quick_env_bench.py humanoid:16384 humanoid:4096 shadow-hand:16384 franka-cube-stack:8192 2>&1 | grep env-steps; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "humanoid or sched or step or envs" 2>&1 | tail -1
