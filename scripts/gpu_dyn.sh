#!/bin/bash
# dynamic vs static B32 work distribution, serial vs pipelined steps, C2/C4/C3; rc n=256 after the TRSM fix
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cs_apply or hash or partition or ms_apply" 2>&1 | tail -2
for c in c2 c4 c3; do
  for dyn in 1 0; do
    for pp in "" "--no-pipeline"; do
      CSK_DYN=$dyn timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-ls --no-extra --no-ne --no-acc $pp > gpurun_out/dyn.json 2> gpurun_out/dyn.err
      python -c "import json; d=json.load(open('gpurun_out/dyn.json')); r=d['roofline']; print('$c dyn=$dyn ${pp:-piped}', 'step', round(d['ms_per_step'],4), 'cs', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))" || tail -3 gpurun_out/dyn.err
    done
  done
done
bash scripts/gpu_rc256b.sh
