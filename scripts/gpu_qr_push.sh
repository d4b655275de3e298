# small solve: DSMEM push of V/T to the next panel owner vs L2 staging (CSK_QR_PUSH=0), same box; solver parity
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2508_14209_b200/csrc scripts/qr_wy_prof.cu -o /tmp/qrp -L paper_2508_14209_b200 -lcsk -Xlinker -rpath=$PWD/paper_2508_14209_b200 2>&1 | grep -v warning | head -5
for r in 1 2; do
  for pu in 0 1; do
    CSK_QR_PUSH=$pu python scripts/solve_timing.py 256x128 512x256 300x150 128x64
    for s in "256 128" "512 256"; do CSK_QR_PUSH=$pu /tmp/qrp $s | grep -E "^m=|mean"; done
  done
done > gpurun_out/qr_push_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_solve.py tests/test_gpu_randcholqr.py -q -x -p no:cacheprovider -k "solve or lstsq or rc" > gpurun_out/qr_push_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/qr_push_tests.txt; cat gpurun_out/qr_push_ab.txt
