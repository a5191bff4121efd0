#!/bin/bash
# r02: host overhead around the fused step, humanoid phased schedule A/B, bench, GPU suite
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for t in quadruped quadruped-anymal-obs humanoid; do timeout 300 python tools/step_overhead.py $t 16384 2>&1 | grep us/step; done
for ns in 1 "" 1 ""; do echo "[no_sched=$ns]"; BSIM_NO_SCHED=$ns timeout 600 python tools/quick_step_bench.py --models humanoid --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python - <<'PY'
import json
l = [x for x in open("gpurun_out/bench.log") if x.startswith("{")]
d = json.loads(l[-1])
print(f"value {d['value']/1e6:.2f} M ms {d['ms_per_step']:.4f} kernel_ms {d['roofline']['kernel_ms']:.4f} e2e {d['e2e']['value']/1e6:.2f} M; " + ", ".join(f"{k} {v['value']/1e6:.2f} M" for k, v in d.get('other_configs', {}).items()))
PY
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -20
