"""Measure profiles/ncu_traffic.json (written to gpurun_out/, committed under profiles/): DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of ONE
launch of the dominant cs_apply kernel per workload, from ncu (run on the GPU box).  bench.py reports it
as roofline.traffic.  usage: python scripts/ncu_traffic.py [c2 c4 c3 ...]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNEL = {"f64": "regex:cs_bulk32", "f32": "regex:cs_bulk64f"}


def traffic(shape, dtype):
    args = [shape] + (["f32"] if dtype == "f32" else [])
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none", "-k",
           KERNEL[dtype], "-s", "2", "-c", "1", "--csv", sys.executable, os.path.join(ROOT, "scripts", "cs_time.py"),
           *args]
    out = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, REPS="1")).stdout
    rows = [r for r in csv.reader(io.StringIO(out[out.index('"ID"'):])) if len(r) > 10]
    h = rows[0]
    tot, name = 0.0, ""
    for r in rows[1:]:
        v = float(r[h.index("Metric Value")].replace(",", ""))
        unit = r[h.index("Metric Unit")]
        tot += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        name = r[h.index("Kernel Name")]
    return tot, name


def main():
    path = os.path.join(ROOT, "gpurun_out", "ncu_traffic.json")   # copied to profiles/ after review
    res = {"_source": "scripts/ncu_traffic.py: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none, one launch (the 3rd) of the dominant cs_apply kernel per workload "
                      "(scripts/cs_time.py, variant auto = B)"}
    for shape in sys.argv[1:] or ["c2", "c4", "c3"]:
        for dtype in ("f64", "f32"):
            if dtype == "f32" and shape != "c2":
                continue
            b, name = traffic(shape, dtype)
            key = shape if dtype == "f64" else shape + "_f32"
            e = {"kernel": name[:120], "dram_bytes_per_launch": b}
            res[key] = {"auto": e, "B": e}
            print(key, b, name[:80], flush=True)
    with open(path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
