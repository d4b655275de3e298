nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s1_gputests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/s1_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/s1_bench_c2.json 2> gpurun_out/s1_bench_c2.log; echo "bench c2 rc=$?"
