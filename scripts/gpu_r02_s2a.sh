# round 2 session 2: state check after re-entry — GPU suite, timings, default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in c2 c4 c3; do timeout 300 python scripts/cs_time.py $c ms; done
for c in c2 c4; do timeout 300 python scripts/cs_time.py $c; done
for c in c2 c3; do timeout 300 python scripts/cs_time.py $c f32; done
CSK_MS_OVERLAP=1 timeout 300 python scripts/cs_time.py c3 ms
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s2a_gputests.txt 2>&1
echo "tests rc=$?"
tail -15 gpurun_out/s2a_gputests.txt
timeout 900 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.log
echo "bench rc=$?"
tail -3 gpurun_out/s2a_bench.log
timeout 900 python scripts/variant_table.py 23 > gpurun_out/s2a_variant_table.json 2> gpurun_out/s2a_variant_table.log; echo "vt rc=$?"
