#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2; do for w in 8 7; do for c in c2 c4; do
  CSK_B32=$w timeout 300 python bench.py --config $c --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra --steps 10 > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json; d=json.load(open('gpurun_out/x.json')); r=d['roofline']; print('W=$w', '$c', 'kernel_ms', round(r['kernel_ms'],4))" || tail -n 3 gpurun_out/x.err
done; done; done
