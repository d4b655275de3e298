#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_solve.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_solve.log; tail -3 gpurun_out/pytest_solve.log
for c in c2 c4 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-acc > gpurun_out/bs_$c.json 2> gpurun_out/bs_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bs_$c.json')); print('$c', 'step', round(d['ms_per_step'],3), 'cs', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, d['normal_equations'])" || tail -3 gpurun_out/bs_$c.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'qr_|cs_bulk|Kernel2|gemm' -c 60 --csv --log-file gpurun_out/launches_solve.csv python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu --no-acc --no-ne > /dev/null 2>&1
