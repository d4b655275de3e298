#!/bin/bash
# C3 chunk-width sweep (CSK_CW) and chunk-major threshold (CSK_CM_DIV)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cw in 66 52 44 34 26; do
  for cm in 2 1; do
  CSK_CW=$cw CSK_CM_DIV=$cm timeout 600 python bench.py --config ${CFG:-c3} --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra --steps 10 > gpurun_out/cw.json 2> gpurun_out/cw.err
  python -c "import json; d=json.load(open('gpurun_out/cw.json')); r=d['roofline']; print('cw $cw cm $cm', 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))" || tail -n 3 gpurun_out/cw.err
  done
done
