#!/bin/bash
# pipelined step outliers: stream-ordered pool cross-stream reuse on (default) vs off (CSK_POOL_NODEP=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
run() {
  timeout 600 env $ENVV python bench.py --config $CFG --no-cpu --no-e2e --no-ls --no-extra --no-ne --no-acc --steps 50 --pipeline > gpurun_out/prio.json 2> gpurun_out/prio.err
  python -c "import json; d=json.load(open('gpurun_out/prio.json')); s=d['step_ms_stats']; print('$CFG $ENVV', round(d['ms_per_step'],4), 'median', round(s['median'],4), 'max', round(s['max'],3))" || tail -3 gpurun_out/prio.err
}
for CFG in c3 c4; do
  for i in 1 2 3 4 5; do ENVV=CSK_POOL_NODEP=1 run; ENVV=CSK_POOL_NODEP=0 run; done
done
