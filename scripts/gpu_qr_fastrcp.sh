# small solve: Newton-refined MUFU sqrt/reciprocal per column vs IEEE sqrt/division (CSK_QR_FASTRCP=0); solver parity
for r in 1 2; do
  for f in 0 1; do CSK_QR_FASTRCP=$f python scripts/solve_timing.py 128x64 256x128 512x256 300x150 64x32; done
done > gpurun_out/qr_fastrcp_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_solve.py tests/test_gpu_randcholqr.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "solve or lstsq or rc or c4" > gpurun_out/qr_fastrcp_tests.txt 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/qr_fastrcp_tests.txt; cat gpurun_out/qr_fastrcp_ab.txt | cut -c1-110
