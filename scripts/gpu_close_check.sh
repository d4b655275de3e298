# end-of-session check: the whole -m gpu suite, smoke(), the default bench line and the C4/C3 lines
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c_gputests.txt 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/c_gputests.txt; cp gpurun_out/parity_slack.json gpurun_out/c_parity_slack.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.txt 2>&1; echo "smoke rc=$?"; cat gpurun_out/c_smoke.txt | tail -1
timeout 900 python bench.py > gpurun_out/c_bench_c2.json 2> gpurun_out/c_bench_c2.log; echo "bench c2 rc=$?"
for c in c4 c3; do timeout 900 python bench.py --config $c > gpurun_out/c_bench_$c.json 2> gpurun_out/c_bench_$c.log; echo "bench $c rc=$?"; done
