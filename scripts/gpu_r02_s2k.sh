# round 2 session 2: G-stage segment-count rule (4/2/1 per CTA, >= 24 k-blocks); C2/C4/C3 launch lists and benches
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ms_apply or gstage or ms_lstsq" > gpurun_out/s2k_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2k_tests.txt
for c in c2 c4 c3; do REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2k_ms_launches_$c.csv python scripts/cs_time.py $c ms > /dev/null 2>&1; done
for c in c4 c3; do timeout 900 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/s2k_bench_$c.json 2> gpurun_out/s2k_bench_$c.log; echo "bench $c rc=$?"; done
timeout 900 python bench.py > gpurun_out/s2k_bench_c2.json 2> gpurun_out/s2k_bench_c2.log; echo "bench c2 rc=$?"
