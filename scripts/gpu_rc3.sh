#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_randcholqr.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_rc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rc.log
tail -n 3 gpurun_out/pytest_rc.log
for cfg in "" "CSK_RC_KERNEL=2" "CSK_RC_KERNEL=1"; do
  echo "cfg=$cfg"; env $cfg timeout 300 python scripts/rc_once.py; env $cfg N=64 timeout 300 python scripts/rc_once.py
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_pass_v3 -c 1 -o gpurun_out/prof_rc env REPS=1 python scripts/rc_once.py > gpurun_out/ncu_rc.log 2>&1
