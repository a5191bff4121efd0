#!/bin/bash
# r02: row-schedule sweep (generic / large kernels) A/B vs the one-lane sweep (BSIM_NO_SCHED), fused-tail
# phase clocks before / after the restrict-qualified obs rows, GPU suite, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in phaseclk0 phaseclk; do for t in quadruped quadruped-anymal-obs; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/phase_clocks.py $t 2>&1 | tail -7; done; done
for v in sched "" sched ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/tail_cost.py 16384 2>&1 | grep "flush=True"; done
for ns in 1 "" 1 ""; do echo "[no_sched=$ns]"; BSIM_NO_SCHED=$ns timeout 600 python tools/quick_step_bench.py --models humanoid --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -20
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; tail -c 400 gpurun_out/bench.log
