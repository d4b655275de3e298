#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c2 c4; do for g in cublas splitk; do
  CFG=$c CSK_GSTAGE=$g timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gsn_${c}_${g}.csv python scripts/gstage_once.py > /dev/null 2>&1
done; done
