#!/bin/bash
# rand_cholQR at n = 256 (the TRSM-workspace path): timing and the per-kernel launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
N=256 LOGD=22 REPS=3 timeout 300 python scripts/rc_once.py
N=256 LOGD=22 REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rc256_launches.csv python scripts/rc_once.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(open("gpurun_out/rc256_launches.csv")))
t = collections.defaultdict(float); c = collections.Counter()
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        k = r["Kernel Name"][:70]; t[k] += float(r["Metric Value"]); c[k] += 1
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda kv: -kv[1])[:12]:
    print(f"{v/1e6:9.3f} ms  {c[k]:4d}x  {100*v/tot:5.1f}%  {k}")
PY
