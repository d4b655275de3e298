#!/bin/bash
# First GPU pass: smoke, GPU parity tests, per-variant CountSketch sweep at C2, default bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p, p.multi_processor_count, p.L2_cache_size)" > gpurun_out/devprops.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in S B T L G; do
  timeout 300 python bench.py --variant $v --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -3 gpurun_out/pytest_gpu.log
