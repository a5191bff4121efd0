#!/bin/bash
# r02: full GPU suite (no -x, all failures listed), new-test detail, fp32 parity tables (fast + IEEE), bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_multirank.py -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
tail -8 gpurun_out/pytest_new.log
timeout 900 python tools/parity_table.py --out gpurun_out/parity_fast.json > gpurun_out/parity_fast.log 2>&1; tail -4 gpurun_out/parity_fast.log
BSIM_LIB_VARIANT=ieee timeout 900 python tools/parity_table.py --out gpurun_out/parity_ieee.json > gpurun_out/parity_ieee.log 2>&1; tail -4 gpurun_out/parity_ieee.log
python tools/parity_table.py --render gpurun_out/parity_fast.json gpurun_out/parity_ieee.json --md gpurun_out/r02_parity_fp32.md > gpurun_out/render.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; tail -c 1500 gpurun_out/bench.log
BENCH_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench2.log 2>&1; echo "bench2 rc=$?" >> gpurun_out/bench2.log; tail -c 600 gpurun_out/bench2.log
