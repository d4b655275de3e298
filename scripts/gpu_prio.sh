#!/bin/bash
# pipelined step stability: host bounded to 2 steps ahead vs unbounded vs serial
cd "${GRAFT_REPO_ROOT:-/root/repo}"
run() {
  timeout 600 env $ENVV python bench.py --config $CFG --no-cpu --no-e2e --no-ls --no-extra --no-ne --no-acc --steps 50 $ARG > gpurun_out/prio.json 2> gpurun_out/prio.err
  python -c "import json; d=json.load(open('gpurun_out/prio.json')); print('$CFG $ENVV $ARG', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['step_ms_stats'].items()}, round(d['roofline']['kernel_ms'],4))" || tail -3 gpurun_out/prio.err
}
for CFG in c4 c3 c2; do
  for i in 1 2 3; do ENVV=CSK_HOST_BOUND=1 ARG= run; done
  for i in 1 2; do ENVV=CSK_HOST_BOUND=0 ARG= run; done
  for i in 1 2; do ENVV=CSK_HOST_BOUND=1 ARG=--no-pipeline run; done
done
