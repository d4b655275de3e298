set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
free -g; nproc; lscpu | grep "Model name"
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-ls --no-extra > gpurun_out/r02_c5_n1.json 2> gpurun_out/r02_c5_n1.log
echo rc=$?
tail -5 gpurun_out/r02_c5_n1.log
