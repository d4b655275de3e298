# one-warp panel team (m <= 128, one CTA) vs the 4-warp team (CSK_QR_TEAM=4), same box; then the solver parity tests
for rep in 1 2; do
  CSK_QR_TEAM=4 python scripts/solve_timing.py 32x16 64x32 96x48 128x64
  python scripts/solve_timing.py 32x16 64x32 96x48 128x64
done > gpurun_out/solve_team_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_solve.py tests/test_gpu_randcholqr.py -q -x -p no:cacheprovider -k "solve or lstsq or rc" > gpurun_out/solve_team_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/solve_team_tests.txt; cat gpurun_out/solve_team_ab.txt
