# fp32 wide chunks: 32-row tiles with 2 CTAs per SM (default) vs the 64-row kernel (CSK_F32_ROWS=64), same box
for rep in 1 2; do
  for r in 64 32; do
    for s in c2 c4 c3 n128; do CSK_F32_ROWS=$r python scripts/cs_time.py $s f32; done
  done
done > gpurun_out/f32rows_ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fp32 or f32 or narrow" > gpurun_out/f32rows_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/f32rows_tests.txt
python - <<'PY'
import json
for l in open("gpurun_out/f32rows_ab.txt"):
    if l.startswith("{"):
        d = json.loads(l); print(d["shape"], "%.4f" % d["ms"], "%.0f" % d["gbs"], d["env"])
PY
