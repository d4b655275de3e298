# single-unit grabs in the tail of the B kernels' dynamic schedule (default) vs fixed grabs of 8 (CSK_GRAB_TAIL=0)
for r in 1 2 3; do
  for t in 0 1; do
    for s in c2 c4 c3 n32; do CSK_GRAB_TAIL=$t python scripts/cs_time.py $s; done
    CSK_GRAB_TAIL=$t python scripts/cs_time.py c2 f32
  done
done > gpurun_out/grab_tail_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "b32 or fp32 or narrow or spread or integer" > gpurun_out/grab_tail_tests.txt 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/grab_tail_tests.txt
python - <<'PY'
import json, collections
acc = collections.defaultdict(list)
for l in open("gpurun_out/grab_tail_ab.txt"):
    if l.startswith("{"):
        d = json.loads(l); acc[(d["shape"], d["dtype"], d["env"].get("CSK_GRAB_TAIL"))].append(d["ms"])
for k in sorted(acc): print(k, ["%.4f" % v for v in acc[k]])
PY
