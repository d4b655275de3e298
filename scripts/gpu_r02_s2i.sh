# round 2 session 2: elected straight-line bulk-reduce issue (one lane, SHFL-broadcast destination) vs the
# per-lane waterfall loop (scratch_ab/old = previous commit's build), same box; parity of cs_apply/ms_apply
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "cs_apply or ms_apply or fp32 or hash or c2_full" > gpurun_out/s2i_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2i_tests.txt
for rep in 1 2; do
for c in c2 c4 c3 n32 n16; do
  CSK_PKG_ROOT=scratch_ab/old timeout 300 python scripts/cs_time.py $c
  timeout 300 python scripts/cs_time.py $c
done
for c in c2 c3 n32; do
  CSK_PKG_ROOT=scratch_ab/old timeout 300 python scripts/cs_time.py $c f32
  timeout 300 python scripts/cs_time.py $c f32
done
done
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk64f -s 3 -c 1 -o gpurun_out/s2i_f32_c2 python scripts/cs_time.py c2 f32 > /dev/null 2>&1; echo "ncu f32 rc=$?"
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:cs_bulk32 -s 3 -c 1 -o gpurun_out/s2i_c2 python scripts/cs_time.py c2 > /dev/null 2>&1; echo "ncu c2 rc=$?"
