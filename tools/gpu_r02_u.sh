#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/sanitize
SAN_TIMEOUT=600 bash tools/gpu_sanitize.sh 2>&1 | grep -E "rc=|SUMMARY" | tail -20
timeout 900 python -m pytest tests/test_gpu_envs.py tests/test_gpu_buffers.py tests/test_gpu_randomize.py tests/test_gpu_scale_parity.py tests/test_gpu_dropin.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"task_reset|fk_kernel|set_root|set_dof|refresh_kernel|contact_geometry|collide|scan_kernel|randomize|force|loco_kernel" \
  -c 20 -o gpurun_out/aux_full -f python tools/aux_kernels_drive.py > gpurun_out/aux_drive.log 2>&1; echo "aux ncu rc=$?"
python tools/ncu_summary.py gpurun_out/aux_full.ncu-rep gpurun_out/r02_aux_kernels_ncu.json --envs 16384 \
  --command "ncu --set full -k regex:(aux kernels) python tools/aux_kernels_drive.py" > /dev/null 2>&1
python tools/aux_kernels_md.py gpurun_out/r02_aux_kernels_ncu.json gpurun_out/aux_drive.log > gpurun_out/r02_aux_kernels.md 2>&1; tail -18 gpurun_out/r02_aux_kernels.md | cut -c1-120
