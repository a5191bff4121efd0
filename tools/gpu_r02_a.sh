cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/quick_step_bench.py > gpurun_out/quick.log 2>&1; tail -8 gpurun_out/quick.log
SAN_TIMEOUT=600 bash tools/gpu_sanitize.sh
