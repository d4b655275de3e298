#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "solve or lstsq" > gpurun_out/pytest_qr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_qr.log; tail -15 gpurun_out/pytest_qr.log
echo wy; timeout 300 python scripts/solve_timing.py
echo wy_p4; CSK_QR_WY_P=4 timeout 300 python scripts/solve_timing.py
echo old_cluster; CSK_QR_WY=0 timeout 300 python scripts/solve_timing.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qr_ -o gpurun_out/qr_wy -f python scripts/solve_once.py 128x64 256x128 512x256 > gpurun_out/ncu_qr.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:qr_ --csv python scripts/solve_once.py 128x64 256x128 512x256 2>&1 | grep qr_ | cut -c1-40,150-
