#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in T B S; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'cs_(row|bulk|smem)_kernel' -c 1 \
    -o gpurun_out/prof_c2_$v python bench.py --variant $v --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/ncu_c2_$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'qr_solve_kernel' -c 1 \
    -o gpurun_out/prof_qr python bench.py --variant T --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc > gpurun_out/ncu_qr.log 2>&1
ls -la gpurun_out/*.ncu-rep
