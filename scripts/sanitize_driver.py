"""Every kernel of libcsk at C1-like sizes, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck, tier T4).  Prints one line per call; a sanitizer error shows in its report."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_14209_b200 as csk  # noqa: E402
import synth  # noqa: E402


def cm(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t() if np.ndim(a) == 2 else \
        torch.from_numpy(np.ascontiguousarray(a)).cuda()


def env(**kv):
    for k, v in kv.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


d, n = 8192, 8
A = synth.gaussian_matrix(d, n, seed=2)
b = synth.rhs(A, "hard", seed=2)
Ad, bd = cm(A), cm(b)
plan = csk.cs_plan(d, 128, 1, sort=True)
plan8k = csk.cs_plan(1 << 13, 128, 1)
for v in ("L", "T", "S", "G", "B", "X"):
    csk.cs_apply(plan, Ad, b=bd, variant=v)
    print("cs_apply", v, flush=True)
csk.cs_apply(plan, cm(A.astype(np.float32)), b=cm(b.astype(np.float32)))
csk.cs_apply(plan, cm(A.astype(np.float32)), b=cm(b.astype(np.float32)), variant="B")   # fp32 copies
print("cs_apply fp32", flush=True)
for kb in ("0", "4096"):   # spread SA^T copies off / one per CTA
    env(CSK_SPREAD_KB=kb)
    csk.cs_apply(plan, Ad, b=bd, variant="B")
    env(CSK_SPREAD_KB=None)
print("cs_apply spread", flush=True)
# narrow B instantiations (KJ = 9 / 17, KJF = 5 / 9; 2-3 CTAs per SM) and the warp-per-element fp32
# combine (2^16 rows at k1 = 16: 64 copies), both outputs (column-major SA, ms_apply's row-major Y)
A24 = synth.gaussian_matrix(20011, 24, seed=8)
p24 = csk.cs_plan(20011, 700, 3)
csk.cs_apply(p24, cm(A24), b=cm(A24[:, 1].copy()), variant="B")
csk.cs_apply(p24, cm(A24.astype(np.float32)), b=cm(A24[:, 1].astype(np.float32)), variant="B")
A6 = synth.gaussian_matrix(1 << 16, 6, seed=9, dtype=np.float32)
p16 = csk.cs_plan(1 << 16, 16, 5)
csk.cs_apply(p16, cm(A6), b=cm(A6[:, 0].copy()), variant="B")
csk.ms_apply(p16, 14, cm(A6), b=cm(A6[:, 0].copy()))
print("cs_apply narrow + warp combine", flush=True)
Am = synth.gaussian_matrix(8192, 100, seed=6)   # G-stage with 4 DMMA warps x 32 rows (NT = 7) and 2 M tiles
csk.ms_apply(csk.cs_plan(8192, 4096, 4), 256, cm(Am), b=cm(Am[:, 0].copy()))
print("ms_apply NT=7 MW=4", flush=True)
wide = synth.gaussian_matrix(4096, 129, seed=3)
csk.cs_apply(csk.cs_plan(4096, 256, 2), cm(wide), b=cm(wide[:, 0].copy()))
print("cs_apply 2 chunks", flush=True)
for k, vv in (("CSK_F32ACC", "0"), ("CSK_F32ACC", "1")):   # fp32: fp64 accumulation vs fp32 copies
    env(**{k: vv})
    A32 = synth.gaussian_matrix(1 << 13, 9, seed=6, dtype=np.float32)
    csk.cs_apply(plan8k, cm(A32), b=cm(A32[:, 0].copy()))
    csk.ms_apply(plan8k, 16, cm(A32), b=cm(A32[:, 0].copy()))
    env(**{k: None})
    print("cs_apply fp32", k, vv, flush=True)
for v in ("L", "S", "G", "T", "X"):                    # every variant into the DMMA G-stage
    env(CSK_VARIANT=str(csk.csk.VARIANTS[v]))
    csk.ms_apply(plan, 16, Ad, b=bd)
    env(CSK_VARIANT=None)
    print("ms_apply via", v, flush=True)
Z = csk.ms_apply(plan, 16, Ad, b=bd)
for e in ({}, {"CSK_QR_WY": "0"}, {"CSK_QR_WY": "0", "CSK_QR_SINGLE": "1"}, {"CSK_QR_WY_P": "2"}):
    env(**e)
    csk.ms_solve(Z, n)
    env(**{k: None for k in e})
    print("ms_solve", e, flush=True)
csk.ne_lstsq(Ad, bd)
print("ne_lstsq", flush=True)
for e in ({}, {"CSK_RC_PATH": "0"}):
    env(**e)
    csk.rc_lstsq(plan, 16, Ad, bd)
    env(**{k: None for k in e})
    print("rc_lstsq", e, flush=True)
Aw = synth.gaussian_matrix(2048, 136, seed=4)
csk.rc_lstsq(csk.cs_plan(2048, 4096, 3), 272, cm(Aw), cm(Aw[:, 0].copy()))
print("rc_lstsq wide", flush=True)
As = synth.gaussian_matrix(1 << 13, 3, seed=5)
for e in ({}, {"CSK_SRHT_KERNEL": "2"}):
    env(**e)
    csk.srht_apply(cm(As), 40, 1)
    env(**{k: None for k in e})
    print("srht_apply", e, flush=True)
csk.srht_apply(cm(As), 200, 1)                     # TMA-fed warp kernel (128 < k <= 256)
print("srht_apply k=200", flush=True)
csk.srht_apply(cm(As[:1024]), 20, 1)
print("srht_apply small", flush=True)
csk.gs_lstsq(Ad, bd, 16, 1)
csk.cs_lstsq(plan, Ad, bd)
csk.msh_lstsq(plan, 16, Ad, bd)
torch.cuda.synchronize()
print("gs/cs/msh lstsq done", flush=True)
# hash plans (codes on the fly, wide and narrow-chunk kernels), the G-stage splits, the async solve,
# and the two-stream pipeline pattern of bench.py
hp = csk.cs_plan(d, 128, 5, row0=3, hash=True)
csk.cs_apply(hp, Ad, b=bd)
csk.cs_apply(csk.cs_plan(4096, 1 << 17, 2, hash=True), cm(wide), b=cm(wide[:, 0].copy()))
print("hash plans done", flush=True)
for ctas in ("1", "5", "300"):   # stream-K G-stage splits
    env(CSK_GS_CTAS=ctas)
    Zk = csk.ms_apply(plan, 24, Ad, b=bd)
    env(CSK_GS_CTAS=None)
print("G-stage splits done", flush=True)
s2 = torch.cuda.Stream()
Zs = [csk.ms_apply(plan, 16, Ad, b=bd) for _ in range(2)]
for i in range(4):
    csk.ms_apply(plan, 16, Ad, b=bd, Z=Zs[i & 1])
    ev = torch.cuda.Event()
    ev.record()
    s2.wait_event(ev)
    x, st, r = csk.ms_solve_async(Zs[i & 1], n, stream=s2)
    torch.cuda.current_stream().wait_stream(s2)
torch.cuda.synchronize()
assert int(st.item()) == 0
print("async solve pipeline done", flush=True)
