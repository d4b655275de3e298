# round 2 session 2: full GPU suite, default bench + C4/C3 lines, launch list of the default bench, traffic refresh
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s2h_gputests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/s2h_gputests.txt
timeout 600 python scripts/ncu_traffic.py c2 c4 c3; echo "traffic rc=$?"
timeout 900 python bench.py > gpurun_out/s2h_bench_c2.json 2> gpurun_out/s2h_bench_c2.log; echo "bench rc=$?"
timeout 900 python bench.py --config c4 > gpurun_out/s2h_bench_c4.json 2> gpurun_out/s2h_bench_c4.log; echo "bench c4 rc=$?"
timeout 900 python bench.py --config c3 > gpurun_out/s2h_bench_c3.json 2> gpurun_out/s2h_bench_c3.log; echo "bench c3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2h_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-ls --no-extra --no-c5 > /dev/null 2>&1; echo "launches rc=$?"
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
