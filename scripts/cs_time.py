"""cs_apply / ms_apply at a BASELINE shape, CUDA-event timed (used by the round-2 GPU scripts).
usage: python scripts/cs_time.py c2|c3|c4|c5 [f32] [ms]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("CSK_PKG_ROOT"):   # A/B: another build of the package (e.g. scratch_ab/old), same inputs
    sys.path.insert(0, os.environ["CSK_PKG_ROOT"])
import paper_2508_14209_b200 as csk  # noqa: E402
import synth  # noqa: E402

SHAPES = {"c2": (1 << 24, 64, 8192, 128), "c4": (1 << 23, 128, 32768, 256), "c3": (1 << 22, 256, 131072, 512),
          "c5": (1 << 27, 64, 8192, 128), "n32": (1 << 23, 32, 2048, 64), "n8": (1 << 23, 8, 128, 16), "n16": (1 << 23, 16, 512, 32), "n128": (1 << 22, 128, 32768, 256),
          "n32d21": (1 << 21, 32, 2048, 64), "n32d22": (1 << 22, 32, 2048, 64), "n24": (1 << 23, 24, 1152, 48)}
name = sys.argv[1]
f32 = "f32" in sys.argv[2:]
ms = "ms" in sys.argv[2:]
d, n, k1, k2 = SHAPES[name]
buf = synth.gaussian_matrix_torch(d, n + 1)
if f32:
    b32 = synth.colmajor_empty(torch, d, n + 1, torch.float32, "cuda")
    b32.copy_(buf)
    del buf
    buf = b32
A, b = buf[:, :n], buf[:, n]
plan = csk.cs_plan(d, k1, 1)
out = synth.colmajor_empty(torch, k2 if ms else k1, n + 1, buf.dtype, "cuda")
fn = (lambda: csk.ms_apply(plan, k2, A, b=b, Z=out)) if ms else (lambda: csk.cs_apply(plan, A, b=b, SA=out))
for _ in range(3):
    fn()
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "20"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    fn()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / reps
nbytes = d * (n + 1) * buf.element_size()
print(json.dumps({"shape": name, "dtype": str(buf.dtype), "op": "ms_apply" if ms else "cs_apply", "ms": t,
                  "gbs": nbytes / t / 1e6, "env": {k: v for k, v in os.environ.items() if k.startswith("CSK_")}}))
