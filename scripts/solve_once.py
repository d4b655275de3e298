"""One ms_solve call per listed shape (for ncu captures of the solve kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14209_b200 as csk  # noqa: E402

shapes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[1:] or ["128x64"])]
for m, n in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    Z = torch.randn((n + 1, m), dtype=torch.float64, device="cuda", generator=g).t()
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    csk.ms_solve(Z, n, x=x)
torch.cuda.synchronize()
print("ok")
