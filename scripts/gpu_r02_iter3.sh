set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ms_apply or gauss or ms_lstsq or fp32" > gpurun_out/r02_it3_tests.txt 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/r02_it3_tests.txt
for c in c2 c4 c3; do timeout 300 python scripts/cs_time.py $c ms; done
for c in c2 c3; do timeout 300 python scripts/cs_time.py $c f32; done
for c in c2 c4 c3; do REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ms3_launches_$c.csv python scripts/cs_time.py $c ms > /dev/null 2>&1; done
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/r02_gstage_c3d python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ncu gs rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk64f -s 3 -c 1 -o gpurun_out/r02_f32_c2b python scripts/cs_time.py c2 f32 > /dev/null 2>&1; echo "ncu f32 rc=$?"
