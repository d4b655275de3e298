#!/bin/bash
# library mempool: full GPU tests, then pipelined vs serial stability (50-step runs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
run() {
  timeout 600 python bench.py --config $CFG --no-cpu --no-e2e --no-ls --no-extra --no-ne --no-acc --steps 50 $ARG > gpurun_out/prio.json 2> gpurun_out/prio.err
  python -c "import json; d=json.load(open('gpurun_out/prio.json')); s=d['step_ms_stats']; print('$CFG $ARG', round(d['ms_per_step'],4), 'median', round(s['median'],4), 'max', round(s['max'],3), 'cs', round(d['roofline']['kernel_ms'],4))" || tail -3 gpurun_out/prio.err
}
for CFG in c3 c4 c2; do
  for i in 1 2 3 4; do ARG=--pipeline run; done
  for i in 1 2; do ARG= run; done
done
