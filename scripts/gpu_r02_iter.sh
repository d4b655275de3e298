# round 2 iteration: parity suites (not the full-size / bench ones), G-stage + fp32 CountSketch timing, ncu
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_solve.py tests/test_gpu_randcholqr.py tests/test_gpu_srht.py -x -q -p no:cacheprovider > gpurun_out/r02_it_tests.txt 2>&1
echo "tests rc=$?"; tail -22 gpurun_out/r02_it_tests.txt
for c in c2 c4 c3; do timeout 300 python scripts/cs_time.py $c; timeout 300 python scripts/cs_time.py $c ms; done
for c in c2 c3; do timeout 300 python scripts/cs_time.py $c f32; CSK_F32ACC=0 timeout 300 python scripts/cs_time.py $c f32; timeout 300 python scripts/cs_time.py $c f32 ms; done
for c in c2 c4 c3; do REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ms_launches_$c.csv python scripts/cs_time.py $c ms > /dev/null 2>&1; done
REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cs_f32_launches_c2.csv python scripts/cs_time.py c2 f32 > /dev/null 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/r02_gstage_c3b python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ncu gs rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk64f -s 3 -c 1 -o gpurun_out/r02_f32_c2 python scripts/cs_time.py c2 f32 > /dev/null 2>&1; echo "ncu f32 rc=$?"
