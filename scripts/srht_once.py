"""SRHT at the paper's sketch shape (k = 2n) on C4's [A b] (d=2^23, n=128): kernel time and GB/s."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_14209_b200 as csk
import synth

logd, n = int(os.environ.get("LOGD", "23")), int(os.environ.get("N", "128"))
reps = int(os.environ.get("REPS", "10"))
d = 1 << logd
dev = torch.device("cuda", 0)
buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, dev)
buf.normal_()
A, b = buf[:, :n], buf[:, n]
Y = torch.empty((n + 1, 2 * n), dtype=torch.float64, device=dev).t()
for _ in range(3):
    csk.srht_apply(A, 2 * n, seed=1, b=b, Y=Y)
torch.cuda.synchronize()
csk.profile_enable(True)
for _ in range(reps):
    csk.srht_apply(A, 2 * n, seed=1, b=b, Y=Y)
ms, launches = csk.profile_read()
csk.profile_enable(False)
byts = d * (n + 1) * 8
print(f"srht d=2^{logd} ncols={n+1} k={2*n}: kernel {ms/launches:.4f} ms, {byts/(ms/launches)/1e6:.1f} GB/s")
