#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck (+ initcheck) over the hot
# path's kernels (tools/sanitize_case.py); logs to gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 python tools/sanitize_case.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
done
