# fp64 B32 narrow instantiations (KJ = 9 / 17 with 3 / 2 CTAs per SM) vs the one-CTA kernel, same box
for rep in 1 2; do
  for nr in 0 1; do
    for s in n8 n16 n24 n32 n32d21 n32d22 c2; do CSK_B32_NARROW=$nr python scripts/cs_time.py $s; done
  done
done > gpurun_out/narrow_ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/narrow_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/narrow_tests.txt; cat gpurun_out/narrow_ab.txt | cut -c1-120
