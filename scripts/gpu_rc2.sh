#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_randcholqr.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_rc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rc.log
tail -n 3 gpurun_out/pytest_rc.log
timeout 300 python scripts/rc_once.py
N=64 timeout 300 python scripts/rc_once.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rc_launches.csv env REPS=2 python scripts/rc_once.py > /dev/null 2>&1
python scripts/launch_share.py gpurun_out/rc_launches.csv 3 2>&1 | head -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_pass -c 1 -o gpurun_out/prof_rc env REPS=1 python scripts/rc_once.py > gpurun_out/ncu_rc.log 2>&1
tail -n 2 gpurun_out/ncu_rc.log
