# round 2 session 2: G-stage with dynamically grabbed stream-K segments; pipelined vs serial C3/C4 steps
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ms_apply or gauss or ms_lstsq or gstage" > gpurun_out/s2j_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2j_tests.txt
timeout 600 python scripts/gstage_bench.py c2 c4 c3
for c in c4 c3; do
  timeout 900 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/s2j_bench_$c.json 2> gpurun_out/s2j_bench_$c.log; echo "bench $c rc=$?"
  timeout 900 python bench.py --config $c --no-e2e --no-cpu --no-pipeline > gpurun_out/s2j_bench_${c}_serial.json 2> gpurun_out/s2j_bench_${c}_serial.log; echo "bench $c serial rc=$?"
done
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/s2j_gstage_c3 python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ncu gs rc=$?"
REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2j_ms_launches_c4.csv python scripts/cs_time.py c4 ms > /dev/null 2>&1
REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2j_ms_launches_c2.csv python scripts/cs_time.py c2 ms > /dev/null 2>&1
