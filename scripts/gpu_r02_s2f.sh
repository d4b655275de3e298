# round 2 session 2: G-stage, 4 consumer warps x 32 rows + dedicated producer warp
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ms_apply or gauss or ms_lstsq or gstage or fp32" > gpurun_out/s2f_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2f_tests.txt
timeout 600 python scripts/gstage_bench.py c2 c4 c3
for c in c2 c4 c3; do timeout 300 python scripts/cs_time.py $c ms; done
for c in c2 c3 n8; do timeout 300 python scripts/cs_time.py $c f32; done
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gstage_kernel -s 3 -c 1 -o gpurun_out/s2f_gstage_c3 python scripts/cs_time.py c3 ms > /dev/null 2>&1; echo "ncu gs rc=$?"
