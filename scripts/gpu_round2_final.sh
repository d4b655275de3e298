# Round-2 close-out evidence (run with gpurun from the repo root; outputs in gpurun_out/, copied to profiles/ r02_*):
# the whole -m gpu suite (parity slack), smoke(), bench lines C2 (default) / C4 / C3 / SRHT / rand_cholQR,
# the Figs 3-5 grid, the csk-kernel launch list of the default step, ncu --set full of the C2 CountSketch and
# of the narrow (n = 32) instantiation. (compute-sanitizer is closed on the GPU pool since round 2.)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_gputests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/f_gputests.txt; cp gpurun_out/parity_slack.json gpurun_out/f_parity_slack.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/f_bench_c2.json 2> gpurun_out/f_bench_c2.log; echo "bench c2 rc=$?"
for c in c4 c3 srht rc; do timeout 900 python bench.py --config $c > gpurun_out/f_bench_$c.json 2> gpurun_out/f_bench_$c.log; echo "bench $c rc=$?"; done
timeout 1800 python bench.py --config fig35 > gpurun_out/f_fig35.json 2> gpurun_out/f_fig35.log; echo "fig35 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(cs_|gstage|qr_wy|codes_|gauss|transpose_out)" -c 120 --csv \
    --log-file gpurun_out/f_launches_c2.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-ls --no-extra --no-c5 > /dev/null 2>&1
echo "launches rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk32 -s 3 -c 1 -o gpurun_out/f_ncu_c2_cs python scripts/cs_time.py c2 > /dev/null 2>&1; echo "ncu c2 rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk32 -s 3 -c 1 -o gpurun_out/f_ncu_n32_cs python scripts/cs_time.py n32 > /dev/null 2>&1; echo "ncu n32 rc=$?"
