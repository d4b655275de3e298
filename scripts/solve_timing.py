"""Time ms_solve alone (CUDA events) on random Z of the BASELINE shapes; prints us per call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14209_b200 as csk  # noqa: E402

for m, n in [(128, 64), (256, 128), (512, 256), (16, 8)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    Z = torch.randn((n + 1, m), dtype=torch.float64, device="cuda", generator=g).t()
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        csk.ms_solve(Z, n, x=x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    reps = 20
    for _ in range(reps):
        csk.ms_solve(Z, n, x=x)
    e1.record()
    torch.cuda.synchronize()
    ref = torch.linalg.lstsq(Z[:, :n], Z[:, n:]).solution[:, 0]
    err = float(torch.linalg.norm(Z[:, :n] @ (x - ref)) / torch.linalg.norm(Z[:, n]))
    print(f"m={m} n={n}: {e0.elapsed_time(e1) / reps * 1e3:8.1f} us per ms_solve (incl. sync), fit err {err:.2e}",
          flush=True)
