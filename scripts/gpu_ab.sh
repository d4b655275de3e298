#!/bin/bash
# same-box A/B of the CountSketch kernel: the current library vs the round-1 library (scratch_ab/)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in "" "scratch_ab/libcsk_prev.so"; do
  for c in c2 c4 c3; do
    CSK_LIB_OVERRIDE=$lib timeout 300 python bench.py --config $c --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra --steps 10 > gpurun_out/x.json 2> gpurun_out/x.err
    python -c "import json; d=json.load(open('gpurun_out/x.json')); r=d['roofline']; print('lib=${lib:-current}', '$c', 'kernel_ms', round(r['kernel_ms'],4))" || tail -n 3 gpurun_out/x.err
  done
done; done
