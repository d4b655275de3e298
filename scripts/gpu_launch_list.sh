set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(cs_|gstage|qr_wy|codes_|gauss|transpose_out)" -c 120 --csv --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-ls --no-extra --no-c5 > /dev/null 2>&1
echo "launches rc=$?"
timeout 900 python bench.py --no-pipeline --no-e2e --no-cpu --no-ls --no-extra --no-c5 > gpurun_out/r2_bench_c2_serial.json 2>/dev/null; echo "serial rc=$?"
