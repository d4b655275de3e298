#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c2} --variant B --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --cs-only > gpurun_out/exp_$label.json 2> gpurun_out/exp_$label.err
  python -c "import json; d=json.load(open('gpurun_out/exp_$label.json')); print('$label', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/exp_$label.err
}
run full CSK_NO_TMA=1 CSK_EXP=0
run noreduce CSK_NO_TMA=1 CSK_EXP=1
run noload CSK_NO_TMA=1 CSK_EXP=2
run neither CSK_NO_TMA=1 CSK_EXP=3
