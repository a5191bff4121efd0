#!/bin/bash
# r02 experiment: the star sweep with one copy of the joint rows (pass type at run time, BSIM_STAR_ONE_COPY)
cd "$GRAFT_REPO_ROOT"
for v in "" onecopy "" onecopy; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_env_bench.py quadruped:16384 quadruped:4096 2>&1 | grep env-steps; done
for v in "" onecopy; do echo "[$v bench]"; BSIM_LIB_VARIANT=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e6, d['roofline']['kernel_ms'], d['e2e']['value']/1e6)"; done
