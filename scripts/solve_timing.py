"""Time the small solve on random Z of the BASELINE shapes (k2 = 2n): ms_solve (host sync per call) and
ms_solve_async (stream-ordered, no sync: the kernel chain alone), CUDA events; prints us per call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14209_b200 as csk  # noqa: E402

shapes = [(64, 32), (128, 64), (256, 128), (512, 256), (16, 8)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for m, n in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    Z = torch.randn((n + 1, m), dtype=torch.float64, device="cuda", generator=g).t()
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rs = torch.zeros(1, dtype=torch.float64, device="cuda")
    for _ in range(3):
        csk.ms_solve(Z, n, x=x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    reps = 20
    e0.record()
    for _ in range(reps):
        csk.ms_solve(Z, n, x=x)
    e1.record()
    torch.cuda.synchronize()
    t_sync = e0.elapsed_time(e1) / reps * 1e3
    e0.record()
    for _ in range(reps):
        csk.ms_solve_async(Z, n, x=x, status=st, sk_resid=rs)
    e1.record()
    torch.cuda.synchronize()
    t_async = e0.elapsed_time(e1) / reps * 1e3
    ref = torch.linalg.lstsq(Z[:, :n], Z[:, n:]).solution[:, 0]
    err = float(torch.linalg.norm(Z[:, :n] @ (x - ref)) / torch.linalg.norm(Z[:, n]))
    print(f"m={m} n={n}: {t_sync:8.1f} us ms_solve (incl. sync), {t_async:8.1f} us ms_solve_async, fit err {err:.2e}"
          f" env={ {k: v for k, v in os.environ.items() if k.startswith('CSK_')} }", flush=True)
