#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (profiling aid)
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  q=""; [ $tool != memcheck ] && q="--quick"
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 python tools/sanitize_run.py $q > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY\|Error' gpurun_out/sanitize_$tool.log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY\|sanitize_run ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
