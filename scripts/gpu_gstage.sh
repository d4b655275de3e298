#!/bin/bash
# split-K DMMA G-stage vs cuBLAS: parity, then the C2/C4 step and phase times for both
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ms_apply or gauss or lstsq" -p no:cacheprovider > gpurun_out/pytest_gstage.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gstage.log
tail -n 3 gpurun_out/pytest_gstage.log
for rep in 1 2; do
for c in c2 c4; do
  for g in cublas splitk; do
    CSK_GSTAGE=$g timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-ls --no-extra --no-acc --no-ne > gpurun_out/gs_${c}_${g}.json 2> gpurun_out/gs_$c.err
    python -c "import json; d=json.load(open('gpurun_out/gs_${c}_${g}.json')); p=d.get('phases_ms',{}); print('$c', '$g', 'step', round(d['ms_per_step'],4), 'cs', round(p.get('cs_apply',0),4), 'g', round(p.get('g_stage',0),4), 'solve', round(p.get('solve',0),4))" || tail -n 5 gpurun_out/gs_$c.err
  done
done
done
