#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "solve" > gpurun_out/pytest_qr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_qr.log; tail -2 gpurun_out/pytest_qr.log
for s in "128 64" "256 128" "512 256"; do timeout 60 scripts/qr_wy_prof $s | grep -v "^ \{1,2\}[0-9]"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qr_wy -o gpurun_out/qr_wy2 -f python scripts/solve_once.py 256x128 > gpurun_out/ncu_qr.log 2>&1; tail -1 gpurun_out/ncu_qr.log
