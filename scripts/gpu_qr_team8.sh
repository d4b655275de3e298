# small solve, m > 256: 8-warp panel team vs the 4-warp team (CSK_QR_TEAM=4), same box; solver parity
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2508_14209_b200/csrc scripts/qr_wy_prof.cu -o /tmp/qrp -L paper_2508_14209_b200 -lcsk -Xlinker -rpath=$PWD/paper_2508_14209_b200 2>&1 | grep -v warning | head -5
for r in 1 2; do
  for t in 4 8; do
    CSK_QR_TEAM=$t python scripts/solve_timing.py 512x256 300x150 400x200
    CSK_QR_TEAM=$t /tmp/qrp 512 256 | grep -E "^m=|mean"
  done
done > gpurun_out/qr_team8_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_solve.py tests/test_gpu_randcholqr.py -q -x -p no:cacheprovider -k "solve or lstsq or rc" > gpurun_out/qr_team8_tests.txt 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/qr_team8_tests.txt; cat gpurun_out/qr_team8_ab.txt
