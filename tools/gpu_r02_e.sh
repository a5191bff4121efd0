#!/bin/bash
# r02: TwoSum joint position error -- A/B timing vs round-1 arithmetic (geom0) and double geometry (geom64),
# full GPU suite (new: contact masks at scale, per-quantity contracts), parity tables, bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in geom0 "" geom64 geom0 "" geom64; do
  BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12 --envs 4096,16384 --prec fp32 > gpurun_out/quick_$v.log 2>&1
  echo "variant=[$v]"; grep us/control gpurun_out/quick_$v.log
done
timeout 1500 python -m pytest tests -m gpu -q -rfE -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "ill-conditioned|tie band|FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -40
for v in "" ieee geom0 geom64; do
  BSIM_LIB_VARIANT=$v timeout 900 python tools/parity_table.py --out gpurun_out/parity_${v:-fast}.json > gpurun_out/parity_${v:-fast}.log 2>&1; tail -1 gpurun_out/parity_${v:-fast}.log
done
python tools/parity_table.py --render gpurun_out/parity_fast.json gpurun_out/parity_ieee.json gpurun_out/parity_geom0.json gpurun_out/parity_geom64.json --md gpurun_out/r02_parity_fp32.md > gpurun_out/render.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; tail -c 600 gpurun_out/bench.log
