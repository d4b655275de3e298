"""Experiment: overlap the small solve of batch i with the CountSketch of batch i+1 (two streams).
Prints ms per step for the serial step and the two-stream pipeline (CSK_GRID limits the CountSketch
grid so SMs stay free for the solve's cluster)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_14209_b200 as csk
import synth

cfg = os.environ.get("CFG", "c2")
d, n, k1, k2 = {"c2": (1 << 24, 64, 8192, 128), "c4": (1 << 23, 128, 32768, 256)}[cfg]
steps = 20
dev = torch.device("cuda", 0)
buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, dev)
buf.normal_()
A, b = buf[:, :n], buf[:, n]
plan = csk.cs_plan(d, k1, 1)
Zs = [synth.colmajor_empty(torch, k2, n + 1, torch.float64, dev) for _ in range(2)]
xs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
st = torch.zeros(steps + 8, dtype=torch.int32, device=dev)
s1 = torch.cuda.current_stream()
s2 = torch.cuda.Stream()


def serial(i):
    csk.ms_apply(plan, k2, A, b=b, Z=Zs[0])
    csk.ms_solve_async(Zs[0], n, x=xs[0], status=st[i:i + 1])


def piped(i):
    Z, x = Zs[i & 1], xs[i & 1]
    csk.ms_apply(plan, k2, A, b=b, Z=Z, stream=s1)
    e = torch.cuda.Event()
    e.record(s1)
    s2.wait_event(e)
    csk.ms_solve_async(Z, n, x=x, status=st[i:i + 1], stream=s2)
    e2 = torch.cuda.Event()
    e2.record(s2)
    piped.done[i & 1] = e2


piped.done = [None, None]


def run(fn, label):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    for i in range(steps):
        if fn is piped and piped.done[i & 1] is not None:
            s1.wait_event(piped.done[i & 1])   # Z[i&1] is free once solve i-2 finished
        fn(i)
    s1.wait_stream(s2)
    e1.record(s1)
    torch.cuda.synchronize()
    assert int((st[:steps] != 0).sum()) == 0
    print(f"{cfg} {label} grid={os.environ.get('CSK_GRID', 'auto')}: {e0.elapsed_time(e1) / steps:.4f} ms/step")


run(serial, "serial")
run(piped, "piped")
