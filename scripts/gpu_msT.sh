#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "ms_apply or ms_lstsq" 2>&1 | tail -n 2
for rep in 1 2; do for t in 0 1; do for c in c2 c4 c3; do
  CSK_MS_TRANSPOSE=$t timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra --steps 10 > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json; d=json.load(open('gpurun_out/x.json')); print('T=$t', '$c', 'step', round(d['ms_per_step'],4), 'phases', {k: round(v,4) for k,v in d['phases_ms'].items() if k in ('cs_apply','g_stage','solve')})" || tail -n 3 gpurun_out/x.err
done; done; done
