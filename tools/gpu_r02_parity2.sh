#!/bin/bash
# r02: scale parity (Ant, ANYmal, humanoid) and authored-scene parity with the knife-edge limit
# sensitivity, per-quantity tables for the shipped and IEEE builds
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/p2
timeout 2400 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_pair_shapes.py -q -rfE -s -p no:cacheprovider > gpurun_out/p2/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p2/pytest.log
grep -E "FAILED|passed|failed|rc=|excused|ill-conditioned" gpurun_out/p2/pytest.log | tail -16
timeout 1500 python tools/parity_table.py --out gpurun_out/p2/parity_fast.json > gpurun_out/p2/parity_fast.log 2>&1; tail -1 gpurun_out/p2/parity_fast.log
BSIM_LIB_VARIANT=ieee timeout 1500 python tools/parity_table.py --out gpurun_out/p2/parity_ieee.json > gpurun_out/p2/parity_ieee.log 2>&1; tail -1 gpurun_out/p2/parity_ieee.log
