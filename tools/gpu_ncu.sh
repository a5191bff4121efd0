#!/bin/bash
# Dev harness: one full ncu capture of the Ant step kernel at 16384 envs.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2108_10470_b200.build > /dev/null 2>&1
TAG=${1:-cur}
MODEL=${2:-quadruped}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_kernel" -s 2 -c 1 -o gpurun_out/step_$TAG -f python tools/prof_step.py 16384 fp32 $MODEL > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
