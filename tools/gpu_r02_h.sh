#!/bin/bash
# r02: per-CTA timeline of the fused step (where the task tail's 30-40 us go), row-schedule sweep on the
# sweep warp (humanoid / franka / shadow hand A/B vs BSIM_NO_SCHED), racecheck of the schedule path, GPU suite
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for t in quadruped quadruped-anymal-obs; do BSIM_LIB_VARIANT=phaseclk timeout 300 python tools/cta_timeline.py $t 16384 2>&1 | tail -28; done
for ns in 1 "" 1 ""; do echo "[no_sched=$ns]"; BSIM_NO_SCHED=$ns timeout 600 python tools/quick_step_bench.py --models humanoid --envs 4096,16384 --prec fp32 2>&1 | grep us/control; done
for ns in 1 ""; do echo "[no_sched=$ns]"; BSIM_NO_SCHED=$ns timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ns$ns.log 2>&1; python - <<'PY'
import json,sys,glob
for f in sorted(glob.glob("gpurun_out/bench_ns*.log")):
    pass
PY
done
python - <<'PY'
import json
for ns in ("1", ""):
    l = [x for x in open(f"gpurun_out/bench_ns{ns}.log") if x.startswith("{")]
    if not l: print("no line", ns); continue
    d = json.loads(l[-1])
    print(f"no_sched={ns!r}: value {d['value']/1e6:.2f} M, " + ", ".join(f"{k} {v['value']/1e6:.2f} M" for k, v in d.get('other_configs', {}).items()))
PY
SAN_TOOLS=racecheck SAN_TIMEOUT=600 bash tools/gpu_sanitize.sh 2>&1 | grep -E "racecheck\[|SUMMARY"
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -20
