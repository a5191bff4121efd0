#!/bin/bash
# r02 final capture: GPU suite, smoke, parity tables (shipped + IEEE builds), bench (+ reference arm),
# launch list, ncu of the fused step (bench workload) and the humanoid, sanitizers
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/final gpurun_out/sanitize
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/final/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/final/pytest_gpu.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 900 python tools/parity_table.py --out gpurun_out/final/parity_fast.json > gpurun_out/final/parity_fast.log 2>&1; tail -1 gpurun_out/final/parity_fast.log
BSIM_LIB_VARIANT=ieee timeout 900 python tools/parity_table.py --out gpurun_out/final/parity_ieee.json > gpurun_out/final/parity_ieee.log 2>&1; tail -1 gpurun_out/final/parity_ieee.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/final/bench_ref.log
python - <<'PY'
import json
d = json.loads([x for x in open("gpurun_out/final/bench.log") if x.startswith("{")][-1])
r = json.loads([x for x in open("gpurun_out/final/bench_ref.log") if x.startswith("{")][-1])
print(f"value {d['value']/1e6:.2f} M ms {d['ms_per_step']:.4f} kernel_ms {d['roofline']['kernel_ms']:.4f} e2e {d['e2e']['value']/1e6:.2f} M clocks {d['clocks']}; " + ", ".join(f"{k} {x['value']/1e6:.2f} M" for k, x in d.get('other_configs', {}).items()))
print("reference arm:", r.get("value"), "same config:", r.get("config") == d.get("config"), "e2e ratio", d['e2e']['value'] / r['value'])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/final/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_kernel" -s 6 -c 1 -o gpurun_out/final/step_full -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/final/ncu_full.log 2>&1; echo "step ncu rc=$?"
python tools/ncu_summary.py gpurun_out/final/step_full.ncu-rep gpurun_out/final/r02_step_${VER:-v34}_ncu.json --envs 16384 --command "ncu --set full -k regex:step_kernel -s 6 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs" > /dev/null 2>&1
SAN_TIMEOUT=600 bash tools/gpu_sanitize.sh 2>&1 | grep -E "rc=|SUMMARY" | tail -20
