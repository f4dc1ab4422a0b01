#!/bin/bash
# compute-sanitizer over the hot path's kernels (tools/sanitize_case.py);
# log to gpurun_out/sanitize_<tool>.log. ONE tool per gpurun call
# (B200_PROFILING.md: several tools in one call have left a GPU unusable):
#   gpurun -- bash tools/sanitize.sh memcheck      (then racecheck, synccheck, initcheck)
tool=${1:-memcheck}
mkdir -p gpurun_out
extra=""
[ $tool = racecheck ] && extra="--racecheck-report all"
[ $tool = memcheck ] && extra="--leak-check full"
timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 python tools/sanitize_case.py \
  > gpurun_out/sanitize_$tool.log 2>&1
echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
