#!/bin/bash
# Per-variant CountSketch sweep at a config (default c2), then the default bench and an ncu launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${1:-c2}
for v in ${VARIANTS:-S B T L G}; do
  timeout 300 python bench.py --config $CFG --variant $v --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${CFG}_$v.json 2> gpurun_out/bench_${CFG}_$v.err
done
if [ -z "$NO_DEFAULT" ]; then
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
fi
