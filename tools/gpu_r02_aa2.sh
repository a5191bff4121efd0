#!/bin/bash
# r02: the Ant analog's 32 x 256 star CTA (ShapeT) -- GPU suite + timing
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/quick_env_bench.py quadruped:16384 quadruped:4096 quadruped-anymal-obs:16384 humanoid:16384 2>&1 | grep env-steps; done
