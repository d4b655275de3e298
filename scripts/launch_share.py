"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

usage: python scripts/launch_share.py launches.csv [steps]
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
    k = r[ki].split("(")[0][:70]
    tot[k] += v * scale
    cnt[k] += 1
T = sum(tot.values())
print(f"{len(rows) - 1} launches, {T / 1e3:.3f} ms of kernel time over {steps} step(s): "
      f"{T / 1e3 / steps:.3f} ms per step (serialised, cold-cache ncu replay)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {100 * v / T:5.1f}%  {v / cnt[k]:9.1f} us/launch  x{cnt[k]:3d}  {k}")
