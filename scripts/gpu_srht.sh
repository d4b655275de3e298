#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_srht.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_srht.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_srht.log
tail -n 20 gpurun_out/pytest_srht.log
timeout 300 python scripts/srht_once.py
N=64 LOGD=24 timeout 300 python scripts/srht_once.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srht_warp -c 1 -o gpurun_out/prof_srht env REPS=1 python scripts/srht_once.py > gpurun_out/ncu_srht.log 2>&1
tail -n 2 gpurun_out/ncu_srht.log
