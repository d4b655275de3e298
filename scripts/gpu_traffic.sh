#!/bin/bash
# dram bytes of the dominant CountSketch launch at C4 and C3 (roofline.traffic), and the e2e line of C2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c4 c3; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cs_bulk32 -c 1 --csv --log-file gpurun_out/traffic_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --no-ls --no-extra --cs-only > /dev/null 2>&1
  grep -E "dram__bytes|gpu__time" gpurun_out/traffic_$c.csv | awk -F'","' '{print "'$c'", $(NF-2), $(NF-1), $NF}'
done
timeout 900 python bench.py --no-cpu --no-ne --no-acc --no-ls --no-extra --steps 5 > gpurun_out/e2e.json 2> gpurun_out/e2e.err
python -c "import json; d=json.load(open('gpurun_out/e2e.json')); print('e2e', d['e2e'])"
