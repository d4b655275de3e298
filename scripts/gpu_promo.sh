#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for p in 128 256 0; do
  CSK_L2PROMO=$p timeout 300 python bench.py --variant B --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/bench_promo_$p.json 2> gpurun_out/bench_promo_$p.err
  python -c "import json; d=json.load(open('gpurun_out/bench_promo_$p.json')); print('B promo $p', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/bench_promo_$p.err
done
CSK_L2PROMO=128 timeout 300 python bench.py --variant X --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/bench_X.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_X.json')); print('X', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cs_bulk_tma_kernel -c 1 -o gpurun_out/prof_c2_B2 python bench.py --variant B --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/ncu_B2.log 2>&1
