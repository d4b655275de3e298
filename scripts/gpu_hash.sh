#!/bin/bash
# CSK_PLAN_HASH A/B: parity of the on-the-fly kernel, then stored vs hashed codes at C2/C4/C3,
# interleaved twice on the same box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "hash or codes or partition" > gpurun_out/pytest_hash.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_hash.log
tail -n 3 gpurun_out/pytest_hash.log
for rep in 1 2; do
for c in c2 c4 c3; do
  for h in "" "--hash-plan"; do
    timeout 600 python bench.py --config $c --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra $h > gpurun_out/hash_$c$h.json 2> gpurun_out/hash_$c.err
    python -c "import json; d=json.load(open('gpurun_out/hash_$c$h.json')); r=d['roofline']; print('$c', '${h:-stored}', 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4), 'step_ms', round(d['ms_per_step'],4))" || tail -n 5 gpurun_out/hash_$c.err
  done
done
done
