#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "cs_apply or worked or identity or partition" > gpurun_out/pytest_b32.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b32.log; tail -2 gpurun_out/pytest_b32.log
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c2} --variant B --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --cs-only > gpurun_out/b32_$label.json 2> gpurun_out/b32_$label.err
  python -c "import json; d=json.load(open('gpurun_out/b32_$label.json')); print('$label', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/b32_$label.err
}
for w in 8 6 4 0; do run w$w CSK_NO_TMA=1 CSK_B32=$w; done
run w8_noreduce CSK_NO_TMA=1 CSK_B32=8 CSK_EXP=1
run w8_noload CSK_NO_TMA=1 CSK_B32=8 CSK_EXP=2
run w6_noreduce CSK_NO_TMA=1 CSK_B32=6 CSK_EXP=1
