#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool initcheck --print-limit 100000 python scripts/sanitize_driver.py > gpurun_out/initcheck_full.txt 2>&1
grep -E "^=========     at " gpurun_out/initcheck_full.txt | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -20
grep -E "ERROR SUMMARY" gpurun_out/initcheck_full.txt
