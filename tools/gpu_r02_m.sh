#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for t in quadruped quadruped-anymal-obs; do BSIM_LIB_VARIANT=resetclk timeout 300 python tools/reset_clocks.py $t 2>&1 | tail -8; done
timeout 300 python tools/step_overhead.py quadruped 16384 2>&1 | grep us/step
timeout 900 python -m pytest tests/test_gpu_envs.py tests/test_gpu_scale_parity.py tests/test_gpu_parallel.py tests/test_gpu_franka_env.py tests/test_gpu_shadow_env.py tests/test_gpu_randomize.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 --no-other-configs > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python - <<'PY'
import json
l = [x for x in open("gpurun_out/bench.log") if x.startswith("{")]
d = json.loads(l[-1])
print(f"value {d['value']/1e6:.2f} M ms {d['ms_per_step']:.4f} kernel_ms {d['roofline']['kernel_ms']:.4f} e2e {d['e2e']['value']/1e6:.2f} M")
PY
