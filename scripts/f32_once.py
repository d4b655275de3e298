"""cs_apply on fp32 C2 ([A b] d=2^24, 65 cols, k1=8192) and on fp64 with odd lda (the 16-row kernel): ms per call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_14209_b200 as csk
import synth

d, n, k1 = 1 << 24, 64, 8192
dev = torch.device("cuda", 0)
plan = csk.cs_plan(d, k1, 1)
for label, dt, pad in (("fp32", torch.float32, 0), ("fp64 lda odd", torch.float64, 1)):
    buf = torch.empty((n + 1, d + pad), dtype=dt, device=dev).t()[:d]
    buf.normal_()
    A, b = buf[:, :n], buf[:, n]
    SA = None
    for _ in range(3):
        SA = csk.cs_apply(plan, A, b=b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        csk.cs_apply(plan, A, b=b, SA=SA)
    e1.record()
    torch.cuda.synchronize()
    print(f"{os.environ.get('CSK_LIB_OVERRIDE') or 'current'} {label}: {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)
    del buf
