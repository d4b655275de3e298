"""G-stage (a5) alone at the BASELINE shapes: the hand-written DMMA kernel inside ms_apply (ms_apply time
minus cs_apply time, CUDA events) against cuBLAS DGEMM (torch.matmul) on the same operand shapes."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2508_14209_b200 as csk  # noqa: E402
import synth  # noqa: E402

SHAPES = {"c2": (1 << 24, 64, 8192, 128), "c4": (1 << 23, 128, 32768, 256), "c3": (1 << 22, 256, 131072, 512)}


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for name in sys.argv[1:] or list(SHAPES):
    d, n, k1, k2 = SHAPES[name]
    buf = synth.gaussian_matrix_torch(d, n + 1)
    A, b = buf[:, :n], buf[:, n]
    plan = csk.cs_plan(d, k1, 1)
    Z = synth.colmajor_empty(torch, k2, n + 1, torch.float64, "cuda")
    SA = synth.colmajor_empty(torch, k1, n + 1, torch.float64, "cuda")
    t_ms = timed(lambda: csk.ms_apply(plan, k2, A, b=b, Z=Z))
    t_cs = timed(lambda: csk.cs_apply(plan, A, b=b, SA=SA))
    G = torch.randn(k2, k1, dtype=torch.float64, device="cuda")
    SAr = torch.randn(k1, n + 1, dtype=torch.float64, device="cuda")
    t_blas = timed(lambda: torch.matmul(G, SAr))
    flops = 2.0 * k2 * k1 * (n + 1)
    g = t_ms - t_cs
    out[name] = {"ms_apply_ms": t_ms, "cs_apply_ms": t_cs, "gstage_ms": g, "gstage_tflops": flops / g / 1e9,
                 "cublas_dgemm_ms": t_blas, "cublas_tflops": flops / t_blas / 1e9}
    print(name, json.dumps(out[name]), flush=True)
    del buf, A, b, G, SAr
    torch.cuda.empty_cache()
