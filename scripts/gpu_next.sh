#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sketch_solve.py tests/test_gpu_srht.py tests/test_gpu_randcholqr.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_next.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_next.log
tail -n 25 gpurun_out/pytest_next.log
timeout 900 python bench.py --config c2 --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-extra --steps 3 --warmup 3 > gpurun_out/ls.json 2> gpurun_out/ls.err
python -c "
import json; d=json.load(open('gpurun_out/ls.json'))
for k,v in d['ls_c4'].items(): print(k, {x: (round(v[x],4) if isinstance(v[x], float) else v[x]) for x in v if x.endswith('_ms') or 'resid' in x or 'status' in x})" || tail -n 20 gpurun_out/ls.err
