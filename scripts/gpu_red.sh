#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c2} --variant B --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --cs-only > gpurun_out/red_$label.json 2> gpurun_out/red_$label.err
  python -c "import json; d=json.load(open('gpurun_out/red_$label.json')); print('$label', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/red_$label.err
}
run base
run neither CSK_EXP=3
run noload CSK_EXP=2
run align128 CSK_LC_ALIGN=16
run align128_noload CSK_LC_ALIGN=16 CSK_EXP=2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cs_bulk32 -c 1 -o gpurun_out/prof_b32_noload env CSK_EXP=2 python bench.py --variant B --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --cs-only > gpurun_out/ncu_b32n.log 2>&1
