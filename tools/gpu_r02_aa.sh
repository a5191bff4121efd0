#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_kernel" -s 2 -c 1 -o gpurun_out/step_humanoid -f python tools/prof_step.py 16384 fp32 humanoid > gpurun_out/ncu_hum.log 2>&1; echo "humanoid ncu rc=$?"
python tools/ncu_summary.py gpurun_out/step_humanoid.ncu-rep gpurun_out/r02_humanoid_step_ncu.json --envs 16384 --command "ncu --set full -k regex:step_kernel -s 2 -c 1 python tools/prof_step.py 16384 fp32 humanoid" > /dev/null 2>&1
python tools/ncu_lines.py gpurun_out/step_humanoid.ncu-rep 30 > gpurun_out/hum_lines.txt 2>&1; head -34 gpurun_out/hum_lines.txt
