"""One ms_apply at C2 or C4 shape (for ncu launch lists of the G-stage kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_14209_b200 as csk
import synth

cfg = os.environ.get("CFG", "c2")
d, n, k1, k2 = {"c2": (1 << 24, 64, 8192, 128), "c4": (1 << 23, 128, 32768, 256)}[cfg]
dev = torch.device("cuda", 0)
buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, dev)
buf.normal_()
plan = csk.cs_plan(d, k1, 1)
Z = synth.colmajor_empty(torch, k2, n + 1, torch.float64, dev)
for _ in range(3):
    csk.ms_apply(plan, k2, buf[:, :n], b=buf[:, n], Z=Z)
torch.cuda.synchronize()
