#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (run on the GPU box); logs -> gpurun_out/sanitize_<tool>.log
for tool in ${@:-memcheck racecheck synccheck}; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
