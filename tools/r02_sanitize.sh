#!/bin/bash
# compute-sanitizer over the small solves of tools/sanitize.py (logs -> gpurun_out/sanitize_<tool>.log)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
     python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
