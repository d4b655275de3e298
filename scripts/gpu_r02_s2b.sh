# round 2 session 2: ncu of the fp32 kernel, the small-k1 contention case, the C3 G-stage, and the overlap launch list
set -x
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk64f -s 3 -c 1 -o gpurun_out/s2b_f32_c2 python scripts/cs_time.py c2 f32 > /dev/null 2>&1; echo "ncu f32 rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk32 -s 3 -c 1 -o gpurun_out/s2b_n16 python scripts/cs_time.py n16 > /dev/null 2>&1; echo "ncu n16 rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/s2b_gstage_c3 python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ncu gs rc=$?"
REPS=2 CSK_MS_OVERLAP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2b_ovl_launches_c3.csv python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ovl rc=$?"
REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2b_ms_launches_c3.csv python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ms rc=$?"
REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2b_f32_launches_c2.csv python scripts/cs_time.py c2 f32 > /dev/null 2>&1; echo "f32 rc=$?"
