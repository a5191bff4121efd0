#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -12
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"task_reset|fk_kernel|set_root|set_dof|refresh_kernel|contact_geometry|collide|scan_kernel|randomize|force|loco_kernel" \
  -c 20 -o gpurun_out/aux_full -f python tools/aux_kernels_drive.py > gpurun_out/aux_drive.log 2>&1; echo "aux ncu rc=$?"
python tools/ncu_summary.py gpurun_out/aux_full.ncu-rep gpurun_out/r02_aux_kernels_ncu.json --envs 16384 \
  --command "ncu --set full -k regex:(aux kernels) python tools/aux_kernels_drive.py" > /dev/null 2>&1
python tools/aux_kernels_md.py gpurun_out/r02_aux_kernels_ncu.json gpurun_out/aux_drive.log > gpurun_out/r02_aux_kernels.md 2>&1; tail -18 gpurun_out/r02_aux_kernels.md
SAN_ENVS=20 SAN_ONLY=envs,buffers,dr timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_drive.py 2>&1 | tail -1
SAN_ENVS=20 SAN_ONLY=envs,buffers,dr timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_drive.py 2>&1 | tail -1
