#!/bin/bash
# Quick iteration: GPU parity tests (optionally filtered by $K), then the CountSketch-only
# bench lines for the configs in $CFGS (default c2 c4 c3).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
for c in ${CFGS:-c2 c4 c3}; do
  timeout 600 python bench.py --config $c --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra > gpurun_out/cs_$c.json 2> gpurun_out/cs_$c.err
  python -c "import json; d=json.load(open('gpurun_out/cs_$c.json')); r=d['roofline']; print('$c', 'kernel_ms', round(r['kernel_ms'],4), 'GB/s', round(r['achieved'],1), 'frac', round(r['frac'],4))" || tail -n 5 gpurun_out/cs_$c.err
done
