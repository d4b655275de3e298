#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "solve or lstsq or gauss or ms_apply" > gpurun_out/pytest_qr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_qr.log; tail -2 gpurun_out/pytest_qr.log
echo blocked; timeout 300 python scripts/solve_timing.py
echo blocked_P4; CSK_QR_P=4 timeout 300 python scripts/solve_timing.py
echo unblocked; CSK_QR_UNBLOCKED=1 timeout 300 python scripts/solve_timing.py
echo single; CSK_QR_UNBLOCKED=1 CSK_QR_SINGLE=1 timeout 300 python scripts/solve_timing.py
