"""fp32 CountSketch at C2 timed in the bench's order (fp64 [A b] resident, a second fp64 buffer, then the
fp32 copy) vs alone -- diagnoses the bench's cs_apply_input_families gaussian_f32 number."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14209_b200 as csk  # noqa: E402
import synth  # noqa: E402

d, n, k1 = 1 << 24, 64, 8192
dev = torch.device("cuda", 0)


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


plan = csk.cs_plan(d, k1, 1)
mode = sys.argv[1] if len(sys.argv) > 1 else "bench"
keep = []
if mode == "bench":
    buf = synth.gaussian_matrix_torch(d, n + 1)
    SA = synth.colmajor_empty(torch, k1, n + 1, torch.float64, "cuda")
    t64 = timed(lambda: csk.cs_apply(plan, buf[:, :n], b=buf[:, n], SA=SA))
    buf2 = synth.colmajor_empty(torch, d, n + 1, torch.float64, dev)
    buf2.copy_(buf)
    t64b = timed(lambda: csk.cs_apply(plan, buf2[:, :n], b=buf2[:, n], SA=SA))
    del buf2
    keep = [buf]
    print(json.dumps({"f64": t64, "f64_second_buffer": t64b}))
src = keep[0] if keep else synth.gaussian_matrix_torch(d, n + 1)
b32 = synth.colmajor_empty(torch, d, n + 1, torch.float32, dev)
b32.copy_(src)
SA32 = synth.colmajor_empty(torch, k1, n + 1, torch.float32, "cuda")
t32 = timed(lambda: csk.cs_apply(plan, b32[:, :n], b=b32[:, n], SA=SA32))
print(json.dumps({"mode": mode, "f32_ms": t32, "mem_GB": torch.cuda.memory_allocated() / 1e9}))
