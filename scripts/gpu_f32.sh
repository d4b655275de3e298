#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "fp32" 2>&1 | tail -n 4
for acc in 1 0; do
  CSK_F32ACC=$acc timeout 600 python bench.py --config c2 --no-cpu --no-e2e --no-ne --no-acc --no-ls --steps 10 > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json; d=json.load(open('gpurun_out/x.json')); print('f32acc=$acc', d['cs_apply_input_families'])" || tail -n 3 gpurun_out/x.err
done
