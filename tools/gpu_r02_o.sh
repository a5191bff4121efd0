#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in noskip ""; do echo "[$v]"; BSIM_LIB_VARIANT=$v timeout 300 python tools/quick_step_bench.py --models quadruped,quadruped12,humanoid --envs 16384 --prec fp32 2>&1 | grep us/control; done
for v in noskip ""; do BSIM_LIB_VARIANT=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1; python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/bench_{v}.log") if x.startswith("{")]
d = json.loads(l[-1])
print(f"[{v}] value {d['value']/1e6:.2f} M; " + ", ".join(f"{k} {x['value']/1e6:.2f} M" for k, x in d.get('other_configs', {}).items()))
PY
done
timeout 1200 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -12
