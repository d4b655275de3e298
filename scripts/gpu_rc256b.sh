#!/bin/bash
# rand_cholQR n = 256 after the TRSM code-size fix: parity (wide cases) + timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_randcholqr.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
N=256 LOGD=22 REPS=3 timeout 300 python scripts/rc_once.py
N=256 LOGD=23 REPS=3 timeout 300 python scripts/rc_once.py
N=200 LOGD=22 REPS=3 timeout 300 python scripts/rc_once.py
N=256 LOGD=22 REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rc256b_launches.csv -k regex:rc_trsm python scripts/rc_once.py > /dev/null 2>&1
grep rc_trsm gpurun_out/rc256b_launches.csv | head -8 | awk -F'","' '{print $NF}'
