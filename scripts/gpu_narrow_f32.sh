# fp32 narrow shapes: B (bulk, fp32 copies) with / without the narrow instantiations and the interleaved
# copies, against T and X (the variants the round-2 table picked for tiny fp32 SA^T); same box
for rep in 1 2; do
  for s in n8 n16 n24 n32 n32d22 c2; do
    CSK_VARIANT=4 CSK_B32_NARROW=0 CSK_SPREAD_KB=0 python scripts/cs_time.py $s f32
    CSK_VARIANT=4 CSK_B32_NARROW=1 CSK_SPREAD_KB=0 python scripts/cs_time.py $s f32
    CSK_VARIANT=4 python scripts/cs_time.py $s f32
    CSK_VARIANT=4 CSK_SPREAD_KB=1024 python scripts/cs_time.py $s f32
    CSK_VARIANT=1 python scripts/cs_time.py $s f32
    CSK_VARIANT=5 python scripts/cs_time.py $s f32
  done
done > gpurun_out/narrow_f32_ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fp32 or f32 or spread or variant" > gpurun_out/narrow_f32_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/narrow_f32_tests.txt
python - <<'PY'
import json
for l in open("gpurun_out/narrow_f32_ab.txt"):
    if l.startswith("{"):
        d = json.loads(l); print(d["shape"], "%.4f" % d["ms"], "%.0f" % d["gbs"], d["env"])
PY
