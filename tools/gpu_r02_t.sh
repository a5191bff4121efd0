#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/san_t
for sec in envs buffers dr; do
  SAN_ENVS=20 SAN_ONLY=$sec timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 400 python tools/sanitize_drive.py > gpurun_out/san_t/racecheck_$sec.log 2>&1
  python tools/racecheck_summary.py gpurun_out/san_t/racecheck_$sec.log | tail -12
done
timeout 900 ncu --set full --clock-control none -k regex:"task_reset|randomize" -c 6 -o gpurun_out/aux_reset -f python tools/aux_kernels_drive.py > gpurun_out/aux_drive2.log 2>&1
python tools/ncu_summary.py gpurun_out/aux_reset.ncu-rep gpurun_out/aux_reset.json --envs 16384 > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/aux_reset.json'))
for m in d['launches']: print(m['kernel'][:50], round(m.get('duration_us',0),1))"
