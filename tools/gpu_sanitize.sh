#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_drive.py
# (racecheck per driver section, hazards summarised by unique site)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
export SAN_ENVS=${SAN_ENVS:-20}
TOOLS=${SAN_TOOLS:-"memcheck racecheck synccheck initcheck"}
for tool in $TOOLS; do
  if [ "$tool" = "racecheck" ]; then
    for sec in envs dr restitution buffers pairs rewards; do
      SAN_ONLY=$sec timeout ${SAN_TIMEOUT:-900} $CS --tool racecheck --racecheck-report all --print-limit 400 \
          --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize/racecheck_$sec.log 2>&1
      echo "racecheck[$sec] rc=$?" >> gpurun_out/sanitize/racecheck_$sec.log
      python tools/racecheck_summary.py gpurun_out/sanitize/racecheck_$sec.log > gpurun_out/sanitize/racecheck_$sec.summary.txt
      tail -3 gpurun_out/sanitize/racecheck_$sec.summary.txt
    done
    continue
  fi
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_drive.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/$tool.log
  tail -3 gpurun_out/sanitize/$tool.log
done
