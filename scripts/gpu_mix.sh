#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c2} --variant B --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --cs-only > gpurun_out/mix_$label.json 2> gpurun_out/mix_$label.err
  python -c "import json; d=json.load(open('gpurun_out/mix_$label.json')); print('$label', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/mix_$label.err
}
for m in 100 48 40 34 32 24 16; do run mix$m CSK_NO_TMA=1 CSK_MIX=$m; done
run mix34_noload CSK_NO_TMA=1 CSK_MIX=34 CSK_EXP=2
run b2_full CSK_B2CFG=1
