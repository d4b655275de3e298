#!/bin/bash
# ncu --set full of the CountSketch main kernel at C4 and C3 (the LS and multisketch configs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c4 c3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'cs_(bulk|tma|row)' -c 1 -o gpurun_out/prof_${c}_main -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --no-ls --no-extra --cs-only > gpurun_out/ncu_main_$c.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_${c}_main.ncu-rep > gpurun_out/ncu_${c}_main.txt 2>&1
done
