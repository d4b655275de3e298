#!/bin/bash
# copy the judged evidence of a scripts/gpu_full.sh pass from gpurun_out/ into profiles/ (round 1 names)
cd "$(dirname "$0")/.."
for c in c2 c3 c4 srht rc; do cp gpurun_out/bench_$c.json profiles/r01_bench_$c.json; done
cp gpurun_out/launches_c2.csv profiles/r01_launches_c2.csv
cp gpurun_out/launch_share_c2.txt profiles/r01_launch_share_c2.txt
python scripts/ncu_summary.py gpurun_out/prof_c2_main.ncu-rep > profiles/r01_ncu_c2_cs_bulk32_final.txt
python scripts/ncu_summary.py gpurun_out/prof_rc.ncu-rep > profiles/r01_ncu_c4_rc_pass.txt
python scripts/ncu_summary.py gpurun_out/prof_srht.ncu-rep > profiles/r01_ncu_c4_srht_warp.txt
python scripts/ncu_summary.py gpurun_out/prof_c3_gstage.ncu-rep > profiles/r01_ncu_c3_gstage_dgemm.txt
