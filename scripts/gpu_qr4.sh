#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qr_ -o gpurun_out/qr_blk128 -f python scripts/solve_once.py 128x64 > gpurun_out/ncu_qr.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qr_ -o gpurun_out/qr_blk512 -f python scripts/solve_once.py 512x256 >> gpurun_out/ncu_qr.log 2>&1
CSK_QR_UNBLOCKED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:qr_ -o gpurun_out/qr_unb512 -f python scripts/solve_once.py 512x256 >> gpurun_out/ncu_qr.log 2>&1
tail -3 gpurun_out/ncu_qr.log
