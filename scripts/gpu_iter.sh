#!/bin/bash
# Iteration: GPU tests, per-variant C2 sweep, optional ncu of a kernel regex.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
CFG=${CFG:-c2}
for v in ${VARIANTS:-X T B S}; do
  timeout 300 python bench.py --config $CFG --variant $v --steps 5 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/bench_${CFG}_$v.json 2> gpurun_out/bench_${CFG}_$v.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${CFG}_$v.json')); print('$v', 'kern_ms', round(d['roofline']['kernel_ms'],3), 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3), 'step_ms', round(d['ms_per_step'],3))" || tail -3 gpurun_out/bench_${CFG}_$v.err
done
if [ -n "$NCU_K" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c 1 \
    -o gpurun_out/prof_${CFG}_${NCU_V} python bench.py --config $CFG --variant ${NCU_V} --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/ncu_${NCU_V}.log 2>&1
fi
