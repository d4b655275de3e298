#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "solve or lstsq or gauss or ms_apply" > gpurun_out/pytest_solve.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_solve.log; tail -2 gpurun_out/pytest_solve.log
run() { local label=$1; shift; local cfg=$1; shift
  env "$@" timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-acc --no-ne > gpurun_out/bs_$label.json 2> gpurun_out/bs_$label.err
  python -c "import json; d=json.load(open('gpurun_out/bs_$label.json')); print('$label', 'step', round(d['ms_per_step'],3), 'cs', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/bs_$label.err
}
run c2 c2
run c4 c4
run c4_cm c4 CSK_CM_DIV=8
run c3 c3
for c in c2 c4 c3; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_step_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-acc --no-ne > /dev/null 2>&1
done
