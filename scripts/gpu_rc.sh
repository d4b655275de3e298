#!/bin/bash
# rand_cholQR: GPU tests + C4 LS comparison (ms / ne / rc) with a chunk-size sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_randcholqr.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_rc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rc.log
tail -n 15 gpurun_out/pytest_rc.log
for ch in "" 16384 131072 1048576; do
  CSK_RC_CHUNK=$ch timeout 600 python bench.py --config c2 --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-extra --steps 5 --warmup 3 > gpurun_out/rc_$ch.json 2> gpurun_out/rc_$ch.err
  python -c "
import json; d=json.load(open('gpurun_out/rc_$ch.json'))
for k,v in d['ls_c4'].items(): print('chunk=$ch', k, {x: v[x] for x in v if x.endswith('_ms') or 'resid' in x or 'status' in x})" || tail -n 5 gpurun_out/rc_$ch.err
done
