# round 2 session 2: look-ahead issue order (CSK_LA) and spread copies (CSK_SPREAD_KB) A/B; fp32; parity of cs_apply/ms_apply
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "cs_apply or ms_apply or fp32 or c2_full or c4_full" > gpurun_out/s2c_tests.txt 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/s2c_tests.txt
for rep in 1 2; do
for c in c2 c4 c3 n32 n16 n8; do
  CSK_LA=0 timeout 300 python scripts/cs_time.py $c
  CSK_LA=1 timeout 300 python scripts/cs_time.py $c
done
done
for c in n32 n16 n8; do for kb in 0 2048 8192 32768; do CSK_SPREAD_KB=$kb timeout 300 python scripts/cs_time.py $c; done; done
for c in c2 c3 n32; do timeout 300 python scripts/cs_time.py $c f32; done
timeout 300 python scripts/cs_time.py c2 f32 ms
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk64f -s 3 -c 1 -o gpurun_out/s2c_f32_c2 python scripts/cs_time.py c2 f32 > /dev/null 2>&1; echo "ncu f32 rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk32 -s 3 -c 1 -o gpurun_out/s2c_c2 python scripts/cs_time.py c2 > /dev/null 2>&1; echo "ncu c2 rc=$?"
