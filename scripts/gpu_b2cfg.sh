#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c2} --variant B --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/b2_$label.json 2> gpurun_out/b2_$label.err
  python -c "import json; d=json.load(open('gpurun_out/b2_$label.json')); print('$label', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3), 'step', round(d['ms_per_step'],3))" || tail -3 gpurun_out/b2_$label.err
}
for c in 0 1 2 3 4; do run cfg$c CSK_B2CFG=$c; done
run noTMA CSK_NO_TMA=1
