"""Measured CountSketch variant table (BASELINE north_star: the variant is picked per (d, n, k1) from
measured HBM GB/s).  Every variant of cs_apply (L, T, S, G, B, X) on [A b] of the paper's shapes
(d x (n + 1), k1 = 2 n^2), fp64 and fp32, CUDA-event timed on the launching stream;
GB/s = algorithmic bytes (A and b read once + SA written once) / time.  Prints one JSON object.

usage: python scripts/variant_table.py [d_log2 ...]      (default 23)"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14209_b200 as csk  # noqa: E402
import synth  # noqa: E402

VARIANTS = ["B", "T", "X", "L", "S", "G"]


def timed(fn, budget_ms=400.0):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    once = e0.elapsed_time(e1)
    reps = int(max(2, min(20, budget_ms / max(once, 1e-3))))
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    logs = [int(a) for a in sys.argv[1:]] or [23]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6548.2
    rows = []
    t0 = time.time()
    for lg in logs:
        d = 1 << lg
        for n in (8, 16, 32, 64, 128, 256):
            k1 = 2 * n * n
            for dt in (torch.float64, torch.float32):
                buf = synth.gaussian_matrix_torch(d, n + 1, dtype=dt)
                A, b = buf[:, :n], buf[:, n]
                plan = csk.cs_plan(d, k1, 1, sort=True)
                SA = synth.colmajor_empty(torch, k1, n + 1, dt, "cuda")
                w = buf.element_size()
                nbytes = d * (n + 1) * w + k1 * (n + 1) * w
                rec = {"d": d, "n": n, "ncols": n + 1, "k1": k1, "dtype": "f64" if dt == torch.float64 else "f32",
                       "ms": {}, "gbs": {}, "frac": {}}
                for v in VARIANTS:
                    if v == "S" and k1 * 8 > 227 * 1024:   # its buckets do not fit shared memory: cs_apply runs B
                        rec["ms"][v] = None
                        rec.setdefault("unsupported", {})[v] = "k1 buckets exceed shared memory (falls back to B)"
                        continue
                    try:
                        ms = timed(lambda: csk.cs_apply(plan, A, b=b, SA=SA, variant=v))
                    except csk.CskError as e:
                        rec["ms"][v] = None
                        rec.setdefault("unsupported", {})[v] = str(e).split(":")[1].strip()
                        continue
                    rec["ms"][v] = ms
                    rec["gbs"][v] = nbytes / ms / 1e6
                    rec["frac"][v] = nbytes / ms / 1e6 / peak
                ok = {v: t for v, t in rec["ms"].items() if t is not None}
                rec["best"] = min(ok, key=ok.get)
                rec["auto_ms"] = timed(lambda: csk.cs_apply(plan, A, b=b, SA=SA))
                rows.append(rec)
                print(json.dumps(rec), file=sys.stderr, flush=True)
                del buf, A, b, plan, SA
                torch.cuda.empty_cache()
    print(json.dumps({"what": "cs_apply variant table", "peak_gbs": peak, "rows": rows,
                      "wall_s": time.time() - t0}))


if __name__ == "__main__":
    main()
