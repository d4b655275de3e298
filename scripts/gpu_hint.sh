#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2; do for h in 0 1; do
  CSK_L2HINT=$h timeout 300 python bench.py --config c3 --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra --steps 10 > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json; d=json.load(open('gpurun_out/x.json')); r=d['roofline']; print('hint=$h c3 kernel_ms', round(r['kernel_ms'],4))" || tail -n 3 gpurun_out/x.err
done; done
CSK_L2HINT=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cs_bulk32 -c 1 --csv --log-file gpurun_out/traffic_c3h.csv python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --no-ls --no-extra --cs-only > /dev/null 2>&1
grep -E "dram__bytes|gpu__time" gpurun_out/traffic_c3h.csv | awk -F'","' '{print "hint", $(NF-2), $(NF-1), $NF}'
