#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "solve or lstsq or gauss or ms_apply" > gpurun_out/pytest_qr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_qr.log; tail -3 gpurun_out/pytest_qr.log
qr() { local label=$1; shift; local c=$1; shift
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'qr_' -c 3 --csv --log-file gpurun_out/lq_$label.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-acc --no-ne --no-ls > /dev/null 2>&1
  grep qr_ gpurun_out/lq_$label.csv | tail -1 | awk -F'","' '{print "'$label'", $(NF)}'
}
qr c2 c2
qr c2_p2 c2 CSK_QR_P=2
qr c2_p4 c2 CSK_QR_P=4
qr c4 c4
qr c4_p4 c4 CSK_QR_P=4
qr c4_p8 c4 CSK_QR_P=8
qr c3 c3
