"""rand_cholQR at C4 (d=2^23, n=128, kappa=1e10): time rc_lstsq with CUDA events (for ncu runs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_14209_b200 as csk
import synth

d, n = 1 << int(os.environ.get("LOGD", "23")), int(os.environ.get("N", "128"))
reps = int(os.environ.get("REPS", "5"))
dev = torch.device("cuda", 0)
buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, dev)
buf[:, :n] = synth.ill_conditioned_torch(d, n, 1e10, seed=2, device=dev)
buf[:, n] = synth.rhs_torch(buf[:, :n], "easy", seed=2)
A, b = buf[:, :n], buf[:, n]
plan = csk.cs_plan(d, 2 * n * n, 1)
x = torch.empty(n, dtype=torch.float64, device=dev)
csk.rc_lstsq(plan, 2 * n, A, b, x=x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    csk.rc_lstsq(plan, 2 * n, A, b, x=x)
e1.record()
torch.cuda.synchronize()
r = float(torch.linalg.norm(b - A @ x) / torch.linalg.norm(b))
print(f"rc_lstsq d=2^{d.bit_length()-1} n={n}: {e0.elapsed_time(e1)/reps:.3f} ms, rel residual {r:.6e}")
