"""Kernel timeline of consecutive cs_apply / ms_apply / pipelined steps at C2 (torch.profiler, CUPTI):
where the time between the CountSketch kernels goes (gaps, G-stage, memsets).
usage: python scripts/step_timeline.py [c2|c4|c3] [f32]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_14209_b200 as csk  # noqa: E402
import synth  # noqa: E402

SHAPES = {"c2": (1 << 24, 64, 8192, 128), "c4": (1 << 23, 128, 32768, 256), "c3": (1 << 22, 256, 131072, 512),
          "n8": (1 << 23, 8, 128, 16), "n16": (1 << 23, 16, 512, 32), "n32": (1 << 23, 32, 2048, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
f32 = "f32" in sys.argv[2:]
d, n, k1, k2 = SHAPES[name]
buf = synth.gaussian_matrix_torch(d, n + 1)
if f32:
    b32 = synth.colmajor_empty(torch, d, n + 1, torch.float32, "cuda")
    b32.copy_(buf)
    del buf
    buf = b32
A, b = buf[:, :n], buf[:, n]
plan = csk.cs_plan(d, k1, 1)
SA = synth.colmajor_empty(torch, k1, n + 1, buf.dtype, "cuda")
Z = synth.colmajor_empty(torch, k2, n + 1, buf.dtype, "cuda")
for _ in range(3):
    csk.ms_apply(plan, k2, A, b=b, Z=Z)
    csk.cs_apply(plan, A, b=b, SA=SA)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

# the bench's pipelined step: ms_apply on the main stream, the solve on a second stream (double-buffered)
s_solve = torch.cuda.Stream()
Zs = [Z, synth.colmajor_empty(torch, k2, n + 1, buf.dtype, "cuda")]
xs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
st = torch.zeros(64, dtype=torch.int32, device="cuda")
rs = torch.zeros(64, dtype=torch.float64, device="cuda")
slot_free = [None, None]
main = torch.cuda.current_stream()


def pipelined(i=[0]):
    sl = i[0] & 1
    if slot_free[sl] is not None:
        slot_free[sl].synchronize()
        main.wait_event(slot_free[sl])
    csk.ms_apply(plan, k2, A, b=b, Z=Zs[sl])
    e = torch.cuda.Event()
    e.record(main)
    s_solve.wait_event(e)
    csk.ms_solve_async(Zs[sl], n, x=xs[sl], status=st[i[0] % 64:i[0] % 64 + 1], sk_resid=rs[i[0] % 64:i[0] % 64 + 1],
                       stream=s_solve)
    e2 = torch.cuda.Event()
    e2.record(s_solve)
    slot_free[sl] = e2
    i[0] += 1


if not f32:   # the solve takes fp64 Z
    for _ in range(4):
        pipelined()
torch.cuda.synchronize()
out = {}
for what, fn in (("cs_apply", lambda: csk.cs_apply(plan, A, b=b, SA=SA)),
                 ("ms_apply", lambda: csk.ms_apply(plan, k2, A, b=b, Z=Z)),
                 ("pipelined_step", pipelined))[: 2 if f32 else 3]:
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(6):
            fn()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    rows = []
    prev_end = None
    for e in ev:
        s, t = e.time_range.start - t0, e.time_range.end - t0
        rows.append({"name": e.name[:60], "start_us": round(s, 1), "dur_us": round(t - s, 1),
                     "gap_us": None if prev_end is None else round(s - prev_end, 1)})
        prev_end = t
    out[what] = rows
    print(what)
    for r in rows:
        print(f"  {r['start_us']:10.1f} {r['dur_us']:9.1f} gap {r['gap_us']}  {r['name']}")
json.dump(out, open("gpurun_out/step_timeline.json", "w"), indent=1)
