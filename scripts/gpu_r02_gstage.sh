# round 2: the hand-written DMMA G-stage -- parity, timing against cuBLAS, L2-reduction microbenchmarks
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ms_apply or gauss or ms_lstsq or hash_plan_ms" > gpurun_out/r02_gs_tests.txt 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/r02_gs_tests.txt
timeout 600 python scripts/gstage_bench.py > gpurun_out/r02_gstage_bench.txt 2>&1; echo "gsbench rc=$?"
cat gpurun_out/r02_gstage_bench.txt
timeout 300 ./scripts/l2red_bench > gpurun_out/r02_l2red.txt 2>&1; echo "l2red rc=$?"
cat gpurun_out/r02_l2red.txt
timeout 600 ncu --set full --import-source on -k regex:gstage_kernel -c 1 -o gpurun_out/r02_gstage_c3 python scripts/gstage_bench.py c3 > /dev/null 2>&1; echo "ncu rc=$?"
