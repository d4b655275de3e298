# fp32 CountSketch: TMA bulk reduce-adds (CSK_F32_RED=0) vs REDG.F32x4 from the LSU (=1), same box,
# interleaved; then the fp32 parity tests with the REDG path forced.
for rep in 1 2; do
  for r in 0 1; do
    for s in c2 c4 c3 n32 n16; do CSK_F32_RED=$r python scripts/cs_time.py $s f32; done
  done
done > gpurun_out/f32red_ab.txt 2>&1
CSK_F32_RED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32 or f32" -p no:cacheprovider > gpurun_out/f32red_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/f32red_tests.txt; cat gpurun_out/f32red_ab.txt
