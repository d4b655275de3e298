# round 2: the whole GPU suite (parity slack recorded) + the default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputests.txt 2>&1
echo "tests rc=$?"
tail -30 gpurun_out/r02_gputests.txt
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.log
echo "bench rc=$?"
tail -3 gpurun_out/r02_bench_default.log
