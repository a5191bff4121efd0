#!/bin/bash
# r02: reset phase clocks, ncu of every non-step kernel, the bench's launch list and one full capture
# of the fused step kernel, compute-sanitizer (memcheck / racecheck / synccheck / initcheck)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in resetclk0 resetclk; do for t in quadruped quadruped-anymal-obs; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/reset_clocks.py $t 2>&1 | tail -8; done; done
for v in prerepack "" prerepack ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/tail_cost.py 16384 2>&1 | grep "flush=True"; done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"task_reset|fk_kernel|set_root|set_dof|refresh_kernel|contact_geometry|collide|scan_kernel|randomize|force|loco_kernel" \
  -c 20 -o gpurun_out/aux_full -f python tools/aux_kernels_drive.py > gpurun_out/aux_drive.log 2>&1; echo "aux ncu rc=$?"; grep -c "==PROF==" gpurun_out/aux_drive.log
python tools/ncu_summary.py gpurun_out/aux_full.ncu-rep gpurun_out/r02_aux_kernels_ncu.json --envs 16384 \
  --command "ncu --set full -k regex:(aux kernels) python tools/aux_kernels_drive.py" > /dev/null 2>&1
python tools/aux_kernels_md.py gpurun_out/r02_aux_kernels_ncu.json gpurun_out/aux_drive.log > gpurun_out/r02_aux_kernels.md 2>&1; head -30 gpurun_out/r02_aux_kernels.md
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_kernel" -s 6 -c 1 -o gpurun_out/step_full -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_full.log 2>&1; echo "step ncu rc=$?"
python tools/ncu_summary.py gpurun_out/step_full.ncu-rep gpurun_out/r02_step_ncu.json --envs 16384 --command "ncu --set full -k regex:step_kernel -s 6 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs" > /dev/null 2>&1
SAN_TIMEOUT=600 bash tools/gpu_sanitize.sh 2>&1 | tail -20
