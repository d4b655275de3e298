# Round-2 GPU evidence in one pass (run with gpurun from the repo root; outputs in gpurun_out/):
#   the whole -m gpu suite (parity slack -> gpurun_out/parity_slack.json), smoke(), the bench lines
#   C2 (default, + c5_n1, ls_c4, cpu_baseline) / C4 / C3, the csk-kernel launch list of the default step,
#   ncu --set full of the dominant kernels, DRAM traffic per launch, the variant table, and the
#   G-stage vs cuBLAS comparison.  Copy what is judged into profiles/ (r02_*).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
free -g; nproc; lscpu | grep "Model name"
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_gputests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.log; echo "bench c2 rc=$?"
for c in c4 c3; do timeout 900 python bench.py --config $c > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.log; echo "bench $c rc=$?"; done
for c in srht rc; do timeout 900 python bench.py --config $c > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.log; echo "bench $c rc=$?"; done
# launch list of the default step (library kernels only: the timed steps, not the input generation)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(cs_|gstage|qr_wy|codes_|gauss|transpose_out)" -c 120 --csv \
    --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-ls --no-extra --no-c5 > /dev/null 2>&1
echo "launches rc=$?"
timeout 600 python scripts/ncu_traffic.py c2 c4 c3; echo "traffic rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk32 -s 3 -c 1 -o gpurun_out/r2_ncu_c2_cs python scripts/cs_time.py c2 > /dev/null 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk64f -s 3 -c 1 -o gpurun_out/r2_ncu_c2_f32 python scripts/cs_time.py c2 f32 > /dev/null 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/r2_ncu_c3_gstage python scripts/cs_time.py c3 ms > /dev/null 2>&1
timeout 600 python scripts/gstage_bench.py c2 c4 c3 > gpurun_out/r2_gstage_bench.txt 2>&1
timeout 900 python scripts/variant_table.py 20 23 > gpurun_out/r2_variant_table.json 2> gpurun_out/r2_variant_table.log; echo "vt rc=$?"
