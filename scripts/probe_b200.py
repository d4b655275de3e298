"""Session probes of the B200: fp64 GEMM rate (cuBLAS via torch), read-only
and copy streaming bandwidth, the shapes of the G-stage and the NE Gram.  Writes
profiles/measured_b200.json.  Library/torch kernels only -- these are denominators, not product."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    out = {"device": torch.cuda.get_device_name(0)}
    p = torch.cuda.get_device_properties(0)
    out["sms"] = p.multi_processor_count
    out["l2_bytes"] = p.L2_cache_size
    # fp64 GEMM 8192^3
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    ms = timed(lambda: a @ a, reps=5)
    out["dgemm_8192_tflops"] = 2 * 8192 ** 3 / ms / 1e9
    # G-stage shapes: (k2 x k1) @ (k1 x ncols)
    for name, (m, k, n) in {"gstage_c2": (128, 8192, 65), "gstage_c3": (512, 131072, 257),
                            "gstage_c4": (256, 32768, 129)}.items():
        G = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
        Y = torch.randn(n, k, dtype=torch.float64, device="cuda").t()
        ms = timed(lambda: G @ Y)
        out[name + "_ms"] = ms
        out[name + "_tflops"] = 2 * m * k * n / ms / 1e9
    del a
    # NE Gram shapes: [A b]^T [A b], d x (n+1)
    for name, (d, nc) in {"gram_c2": (1 << 24, 65), "gram_c4": (1 << 23, 129)}.items():
        A = torch.randn(nc, d, dtype=torch.float64, device="cuda").t()
        ms = timed(lambda: A.t() @ A, reps=5)
        out[name + "_gemm_ms"] = ms
        out[name + "_gemm_tflops"] = 2 * d * nc * nc / ms / 1e9
        del A
    # streaming: read-only (sum) and copy over 8 GiB fp64
    x = torch.empty(1 << 30, dtype=torch.float64, device="cuda").normal_()
    y = torch.empty_like(x)
    ms = timed(lambda: x.sum(), reps=10)
    out["read_sum_8GiB_gbs"] = x.numel() * 8 / ms / 1e6
    ms = timed(lambda: y.copy_(x), reps=10)
    out["copy_8GiB_gbs"] = 2 * x.numel() * 8 / ms / 1e6
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "measured_b200.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    sys.exit(main())
