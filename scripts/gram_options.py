"""Time Gram-matrix options for the normal-equations baseline at the C2 and C4 shapes (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14209_b200 as csk  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for d, n in [(1 << 24, 64), (1 << 23, 128)]:
    nc = n + 1
    buf = torch.randn((nc, d), dtype=torch.float64, device="cuda").t()   # column-major d x nc
    A, b = buf[:, :n], buf[:, n]
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    flops = 2.0 * d * nc * nc
    res = {}
    res["torch mm [A b]^T[A b]"] = timeit(lambda: buf.t() @ buf)
    res["torch mm A^T A"] = timeit(lambda: A.t() @ A)
    for P in (148, 296, 592, 1184):
        rb = d // P
        blocks = buf[: P * rb].t().reshape(nc, P, rb).permute(1, 2, 0)   # P x rb x nc (strided)
        res[f"torch bmm split-K P={P} + sum"] = timeit(lambda: torch.bmm(blocks.transpose(1, 2), blocks).sum(0))
    for mode in ("", "gemm", "syrk"):
        if mode:
            os.environ["CSK_NE_GRAM"] = mode
        else:
            os.environ.pop("CSK_NE_GRAM", None)

        def ne():
            try:
                csk.ne_lstsq(A, b, x=x)
            except csk.CskError:
                pass
        res[f"ne_lstsq gram={mode or 'splitk'} (full solve)"] = timeit(ne, reps=2 if mode else 5)
    os.environ.pop("CSK_NE_GRAM", None)
    print(f"d={d} n={n}: Gram flops {flops / 1e9:.0f} GFLOP (GEMM form)")
    for k, v in res.items():
        print(f"   {k:42s} {v:8.3f} ms   {flops / v / 1e9:6.1f} TF/s(GEMM-form)")
