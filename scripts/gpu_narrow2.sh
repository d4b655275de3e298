# narrow fp64/fp32 kernels + warp-per-element fp32 combine: timings and the parity tests that cover them
for rep in 1 2; do
  for s in n8 n16 n24 n32 n32d21 n32d22 c2; do python scripts/cs_time.py $s; python scripts/cs_time.py $s f32; done
  for s in n8 n16 n32 c2; do python scripts/cs_time.py $s ms; python scripts/cs_time.py $s f32 ms; done
done > gpurun_out/narrow2_ab.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/narrow2_tests.txt 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/narrow2_tests.txt
python - <<'PY'
import json
for l in open("gpurun_out/narrow2_ab.txt"):
    if l.startswith("{"):
        d = json.loads(l); print(d["shape"], d["dtype"][6:], d["op"], "%.4f" % d["ms"], "%.0f" % d["gbs"])
PY
