# rand_cholQR at n = 256 (the Q0-workspace path): parity, timing, launch list, ncu of the TRSM kernel
set -x
timeout 900 python -m pytest tests/test_gpu_randcholqr.py -x -q -p no:cacheprovider > gpurun_out/rcw_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/rcw_tests.txt
LOGD=22 N=256 timeout 300 python scripts/rc_once.py
LOGD=23 N=256 REPS=2 timeout 300 python scripts/rc_once.py
LOGD=22 N=200 timeout 300 python scripts/rc_once.py
LOGD=22 N=256 REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:rc_trsm -s 2 -c 1 -o gpurun_out/rcw_trsm2 python scripts/rc_once.py > /dev/null 2>&1; echo "ncu rc=$?"
