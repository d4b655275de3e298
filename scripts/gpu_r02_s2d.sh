# round 2 session 2: G-stage with a producer warp and full/empty mbarriers (no CTA barrier per k-block)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ms_apply or gauss or ms_lstsq or gstage or spread or cs_apply_fp64" > gpurun_out/s2d_tests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/s2d_tests.txt
timeout 600 python scripts/gstage_bench.py c2 c4 c3
for c in c2 c4 c3 n8 n16; do timeout 300 python scripts/cs_time.py $c ms; done
for c in n8 n16; do timeout 300 python scripts/cs_time.py $c; done
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/s2d_gstage_c3 python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ncu gs rc=$?"
REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2d_ms_launches_c4.csv python scripts/cs_time.py c4 ms > /dev/null 2>&1; echo "l rc=$?"
