# round 2 session 2: fp32 double-buffered tiles A/B (CSK_F32NB), G-stage launch lists at C2/C4, variant table, default bench
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fp32" > gpurun_out/s2g_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2g_tests.txt
for rep in 1 2; do for c in c2 c3 n32; do
  CSK_F32NB=1 timeout 300 python scripts/cs_time.py $c f32
  timeout 300 python scripts/cs_time.py $c f32
done; done
for c in c2 c4; do REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2g_ms_launches_$c.csv python scripts/cs_time.py $c ms > /dev/null 2>&1; done
timeout 900 python scripts/variant_table.py 20 23 > gpurun_out/s2g_variant_table.json 2> gpurun_out/s2g_variant_table.log; echo "vt rc=$?"
timeout 900 python bench.py > gpurun_out/s2g_bench.json 2> gpurun_out/s2g_bench.log; echo "bench rc=$?"
tail -2 gpurun_out/s2g_bench.log
