#!/bin/bash
# compute-sanitizer over every kernel; summaries -> gpurun_out/sanitizer_*.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$? : $(grep -c 'done' gpurun_out/sanitizer_$tool.txt) completions; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_$tool.txt | tail -1)"
done
