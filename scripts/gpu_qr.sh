#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "solve or lstsq or gauss or ms_apply" > gpurun_out/pytest_qr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_qr.log; tail -2 gpurun_out/pytest_qr.log
for c in c2 c4 c3; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'qr_' -c 3 --csv --log-file gpurun_out/launches_qr_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-acc --no-ne > /dev/null 2>&1
grep qr_cluster gpurun_out/launches_qr_$c.csv | tail -1 | awk -F'","' '{print "'$c'", $(NF)}'
done
