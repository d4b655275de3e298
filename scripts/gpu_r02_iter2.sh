# round 2 iteration 2: 16-warp G-stage + parity; variant table
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ms_apply or gauss or ms_lstsq or fp32" > gpurun_out/r02_it2_tests.txt 2>&1
echo "tests rc=$?"; tail -8 gpurun_out/r02_it2_tests.txt
for c in c2 c4 c3; do timeout 300 python scripts/cs_time.py $c ms; done
for c in c2 c4 c3; do REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ms2_launches_$c.csv python scripts/cs_time.py $c ms > /dev/null 2>&1; done
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/r02_gstage_c3c python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ncu gs rc=$?"
timeout 900 python scripts/variant_table.py 23 > gpurun_out/r02_variant_table.json 2> gpurun_out/r02_variant_table.log; echo "vt rc=$?"
tail -3 gpurun_out/r02_variant_table.log
