#!/usr/bin/env python
"""Benchmark of the multisketch sketch-and-solve hot path on B200 (arXiv 2508.14209).

One STEP = one pass of the whole hot path over one batch of synthetic input
(SURVEY 8(a)): CountSketch apply of [A b] (a3) -> Gaussian stage Z = G(S[A b]) (a5)
-> NCCL all-reduce of Z when N > 1 (a6) -> Householder solve (a7).  Codes (a1) and
G (a4) live in the plan (timed separately as plan_ms); the normal-equations
baseline (a8) is timed beside it on the same [A b].

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
  python bench.py --config srht | rc       # the NEXT rows (SRHT, rand_cholQR), one GPU
  python bench.py --config kappa           # Fig 8: residual vs kappa(A) for every solver
  python bench.py --config fig35           # Figs 3-5: sketch / LS times over the paper's (d, n) grid

Rank 0 prints ONE JSON line.  value = whole-job GB/s of [A b] sketched and solved
(sum over ranks of d*(n+1)*8 bytes / max-over-ranks step time).  Weak scaling:
every rank owns a d-row block of the row-partitioned global matrix.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CountSketch apply GB/s (% HBM peak) & multisketch-LS ms vs normal eqns, 1/2/4/8 B200"
CONFIGS = {
    "c1": dict(d=4096, n=8, k1=64, k2=16, kappa=None, name="C1: d=4096 n=8 k1=64 fp64"),
    "c2": dict(d=1 << 24, n=64, k1=8192, k2=128, kappa=None,
               name="C2: CountSketch d=2^24 n=64 (+b) k1=2n^2=8192 k2=2n=128 fp64 col-major, Gaussian A"),
    "c3": dict(d=1 << 22, n=256, k1=131072, k2=512, kappa=None,
               name="C3: multisketch d=2^22 n=256 (+b) k1=131072 k2=512 fp64, Gaussian A"),
    "c4": dict(d=1 << 23, n=128, k1=32768, k2=256, kappa=1e10,
               name="C4: multisketch LS [A b] d=2^23 n=128 k1=32768 k2=256 fp64, kappa(A)=1e10"),
    "c5": dict(d=1 << 27, n=64, k1=8192, k2=128, kappa=None,
               name="C5: row-partitioned d=2^27 n=64 (+b) k1=8192 k2=128 fp64 (strong scaling)"),
}
SKETCH_SEED, DATA_SEED = 1, 2
FALLBACK_HBM_GBS = 6650.0
NOMINAL_HBM_GBS = 8000.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ peaks
def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload_key, variant):
    """dram bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        e = t.get(workload_key, {}).get(str(variant))
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            log(f"[bench] NVML unavailable: {e}")

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def oracle_sample_rows(n, target_s, k1, k2):
    """Rows of an oracle ms_lstsq sample that take about target_s seconds on one core."""
    import numpy as np
    import oracle
    import synth
    d0 = 1 << 15
    A = synth.gaussian_matrix(d0, n, seed=DATA_SEED)
    b = synth.rhs(A, "easy", seed=DATA_SEED)
    t = time.perf_counter()
    h, s = oracle.codes(d0, k1, SKETCH_SEED)
    oracle.cs_apply(h, s, A, k1, b=b)
    per_row = (time.perf_counter() - t) / d0
    t = time.perf_counter()
    G = oracle.gauss(k2, k1, SKETCH_SEED)
    oracle.gemm_comp(G, np.zeros((k1, n + 1)))
    fixed = time.perf_counter() - t
    rows = int(max(1 << 12, (target_s - fixed) / max(per_row, 1e-12)))
    return rows, per_row, fixed


def run_oracle_sample(cfg, rows):
    """Oracle multisketch LS on the first `rows` rows of a host-generated sample of the workload."""
    import oracle
    import synth
    n, k1, k2 = cfg["n"], cfg["k1"], cfg["k2"]
    A = synth.gaussian_matrix(rows, n, seed=DATA_SEED)
    b = synth.rhs(A, "easy", seed=DATA_SEED)
    t = time.perf_counter()
    oracle.ms_lstsq(A, b, k1, k2, SKETCH_SEED)
    return time.perf_counter() - t


# ------------------------------------------------------------- reference arm
def bench_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    n = cfg["n"]
    d = cfg["d"] if args.config != "c5" else cfg["d"] // max(ws, 1)
    total_budget = 150.0
    per_step = max(0.5, min(8.0, total_budget / max(1, args.steps + args.warmup)))
    rows, per_row, fixed = oracle_sample_rows(n, per_step, cfg["k1"], cfg["k2"])
    rows = min(rows, d)
    for _ in range(args.warmup):
        run_oracle_sample(cfg, rows)
    times = [run_oracle_sample(cfg, rows) for _ in range(args.steps)]
    t = statistics.mean(times)
    gbs = rows * (n + 1) * 8 / t / 1e9
    sample = (f"first {rows} rows of the {cfg['name']} workload (host-generated, same shape and "
              f"distribution), full oracle ms_lstsq (codes + CountSketch + G + G-stage + Householder) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "d": d, "n": n, "k1": cfg["k1"], "k2": cfg["k2"],
                   "parallelism": "oracle (CPU, 1 thread)"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cores_available": cpu_cores()},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------- LS comparison
def ls_compare(args, cfg, kappa, dev, stream):
    """Multisketch sketch-and-solve (ms_apply + ms_solve, as in the step) vs the normal
    equations on one [A b] of the cfg shape with condition number kappa; CUDA-event times
    over args.steps calls each, relative residuals ||b - Ax|| / ||b|| against the QR optimum."""
    import torch

    import paper_2508_14209_b200 as csk
    import synth

    d, n, k1, k2 = cfg["d"], cfg["n"], cfg["k1"], cfg["k2"]
    buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, dev)
    buf[:, :n] = synth.ill_conditioned_torch(d, n, kappa, seed=DATA_SEED, device=dev)
    buf[:, n] = synth.rhs_torch(buf[:, :n], "easy", seed=DATA_SEED)
    A, b = buf[:, :n], buf[:, n]
    plan = csk.cs_plan(d, k1, SKETCH_SEED)
    Z = synth.colmajor_empty(torch, k2, n + 1, torch.float64, dev)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def ms():
        csk.ms_apply(plan, k2, A, b=b, Z=Z)
        return csk.ms_solve(Z, n, x=x)[1]

    def ne():
        try:
            csk.ne_lstsq(A, b, x=x)
            return "OK"
        except csk.CskError as e:
            return str(e).split(":")[1].strip()

    def rc():
        try:
            csk.rc_lstsq(plan, k2, A, b, x=x)
            return "OK"
        except csk.CskError as e:
            return str(e).split(":")[1].strip()

    def gs():      # Gaussian sketch-and-solve, k = 2n (Fig 5 "Gaussian" bars)
        return csk.gs_lstsq(A, b, k2, SKETCH_SEED, x=x)[1]

    def cs():      # CountSketch-only sketch-and-solve, k1 = 2n^2 (GEQRF on k1 x (n+1))
        return csk.cs_lstsq(plan, A, b, x=x)[1]

    def msh():     # Count+SRHT multisketch
        return csk.msh_lstsq(plan, k2, A, b, x=x)[1]

    out = {"kappa": kappa, "workload": cfg["name"].replace("kappa(A)=1e10", f"kappa(A)={kappa:.0e}")}
    solvers = [("ms", ms), ("ne", ne), ("rc", rc)]
    if not getattr(args, "no_ls_extra", False):
        solvers += [("gs", gs), ("cs", cs), ("msh", msh)]
    for name, fn in solvers:
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0.record(stream)
        res = [fn() for _ in range(args.steps)]
        e1.record(stream)
        torch.cuda.synchronize()
        out[f"{name}_ms"] = e0.elapsed_time(e1) / args.steps
        if name in ("ne", "rc"):
            out[f"{name}_status"] = res[-1]
        fn()
        out[f"{name}_rel_residual"] = float(torch.linalg.norm(b - A @ x) / torch.linalg.norm(b)) \
            if (name not in ("ne", "rc") or res[-1] == "OK") else None
    R = torch.linalg.qr(buf, mode="r")[1]
    out["true_rel_residual"] = float(abs(R[n, n]) / torch.linalg.norm(b))
    out["speedup_ms_vs_ne"] = out["ne_ms"] / out["ms_ms"]
    # rand_cholQR: the true LS solution; its pass over A is TRSM d n^2 + SYRK-form Gram d n^2 flops
    out["rc_pass_gflop"] = 2.0 * d * n * n / 1e9
    del R, buf, A, b, Z
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- our arm
def bench_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_14209_b200 as csk
    import synth

    ws, rank, local = dist_env()
    # CSK_BENCH_BACKEND=gloo lets the N > 1 logic run with several ranks on one GPU (a test of the
    # partitioning, barriers and max-over-ranks timing; NCCL refuses two ranks on one device)
    backend = os.environ.get("CSK_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    if args.variant != "auto":
        os.environ["CSK_VARIANT"] = str(csk.csk.VARIANTS[args.variant])
    n, k1, k2 = cfg["n"], cfg["k1"], cfg["k2"]
    strong = args.config == "c5"
    d_glob = cfg["d"] if strong else cfg["d"] * ws
    d = d_glob // ws if strong else cfg["d"]
    row0 = rank * d
    ncols = n + 1
    bytes_step = d * ncols * 8                        # [A b] read once per step (per rank)
    stream = torch.cuda.current_stream(dev)

    # ---- inputs: [A b] contiguous column-major (d x (n+1)), resident in HBM before timing
    t0 = time.perf_counter()
    buf = synth.colmajor_empty(torch, d, ncols, torch.float64, dev)
    if cfg["kappa"]:
        buf[:, :n] = synth.ill_conditioned_torch(d, n, cfg["kappa"], seed=DATA_SEED * 1000 + rank, device=dev)
    else:
        buf[:, :n] = synth.gaussian_matrix_torch(d, n, seed=DATA_SEED * 1000 + rank, device=dev)
    buf[:, n] = synth.rhs_torch(buf[:, :n], "easy", seed=DATA_SEED * 1000 + rank)
    A, b = buf[:, :n], buf[:, n]
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: inputs {bytes_step / 1e9:.2f} GB generated in {time.perf_counter() - t0:.1f}s")

    # ---- plan (a1 codes; a4 G is drawn on first use and cached)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    plan = csk.cs_plan(d, k1, SKETCH_SEED, row0=row0, sort=(args.variant == "G"), hash=args.hash_plan)
    ev1.record(stream)
    torch.cuda.synchronize()
    plan_ms = ev0.elapsed_time(ev1)
    Z = synth.colmajor_empty(torch, k2, ncols, torch.float64, dev)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    t = time.perf_counter()
    csk.ms_apply(plan, k2, A, b=b, Z=Z)                 # draws and caches G (k2 x k1)
    torch.cuda.synchronize()
    gauss_first_ms = (time.perf_counter() - t) * 1e3

    SA_ws = synth.colmajor_empty(torch, k1, ncols, torch.float64, dev)

    # a7's numerical status and sketched residual stay on the device (ms_solve_async): one slot per
    # step, all checked after the timed region, so no step drains the GPU with a host sync
    st_buf = torch.zeros(max(args.steps, args.warmup, 1), dtype=torch.int32, device=dev)
    rs_buf = torch.zeros(max(args.steps, args.warmup, 1), dtype=torch.float64, device=dev)

    # Batches are pipelined over two streams (unless --no-pipeline): the small solve of step i (a few
    # CTAs for ~0.1-0.6 ms) runs on its own stream while step i+1's sketch starts; Z and x are
    # double-buffered and slot reuse waits for the solve that last read it.  Every step still runs
    # the whole path on its own batch; the timed region ends after both streams drain.
    pipe = not args.no_pipeline and not args.cs_only
    prio = int(os.environ.get("CSK_SOLVE_PRIO", "0"))   # experiment: solve-stream priority
    host_bound = os.environ.get("CSK_HOST_BOUND", "1") != "0"   # experiment: unbounded host run-ahead
    s_solve = torch.cuda.Stream(device=dev, priority=prio) if pipe else stream
    Zs = [Z, synth.colmajor_empty(torch, k2, ncols, torch.float64, dev)]
    xs = [x, torch.empty(n, dtype=torch.float64, device=dev)]
    slot_free = [None, None]

    def step(i=0):
        if args.cs_only:                                 # kernel experiments: the CountSketch alone
            csk.cs_apply(plan, A, b=b, SA=SA_ws)
            return
        sl = i & 1 if pipe else 0
        if slot_free[sl] is not None:
            if host_bound:
                slot_free[sl].synchronize()   # the host stays <= 2 steps ahead of the device
            stream.wait_event(slot_free[sl])
        csk.ms_apply(plan, k2, A, b=b, Z=Zs[sl])
        if ws > 1:
            dist.all_reduce(Zs[sl].t())                  # a6: NCCL over NVLink (contiguous view of Z)
        if pipe:
            e = torch.cuda.Event()
            e.record(stream)
            s_solve.wait_event(e)
        csk.ms_solve_async(Zs[sl], n, x=xs[sl], status=st_buf[i:i + 1], sk_resid=rs_buf[i:i + 1],
                           stream=s_solve)               # a7
        if pipe:
            e = torch.cuda.Event()
            e.record(s_solve)
            slot_free[sl] = e

    def join():
        if pipe:
            stream.wait_stream(s_solve)

    def check_status(what, count):
        bad = int((st_buf[:count] != 0).sum().item())
        if bad:
            raise RuntimeError(f"{what}: {bad} step(s) returned a singular sketched R")

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if ws == 1:
            return v
        t_ = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        return float(t_.item())

    for i in range(args.warmup):
        step(i)
    barrier()
    check_status("warm-up", args.warmup)
    st_buf.fill_(-1)
    clocks = ClockSampler(local)
    csk.launch_count(reset=True)
    # the dominant kernel (cs_apply main kernel) is timed inside the timed region: the library
    # records a pooled CUDA event on its launching stream right before the launch and one right
    # after it (csk_profile_enable); per-step times come from events around each step
    csk.profile_enable(True)
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    with clocks:
        barrier()
        torch.cuda.nvtx.range_push("csk_timed")   # ncu --nvtx --nvtx-include csk_timed/ (launch list)
        ev0.record(stream)
        for i in range(args.steps):
            step_ev[i][0].record(stream)
            step(i)
            step_ev[i][1].record(stream)
        join()
        ev1.record(stream)
        barrier()
        torch.cuda.nvtx.range_pop()
    if not args.cs_only:
        check_status("timed steps", args.steps)   # every slot written (-1 = not run) and OK
    launches = csk.launch_count() // max(1, args.steps) * args.steps
    step_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    value = ws * bytes_step / (step_ms * 1e-3) / 1e9
    per_step = sorted(a.elapsed_time(b_) for a, b_ in step_ev)
    step_stats = {"median": per_step[len(per_step) // 2], "mean": sum(per_step) / len(per_step),
                  "min": per_step[0], "max": per_step[-1]}
    kern_ms_total, kern_launches = csk.profile_read()
    csk.profile_enable(False)
    kern_ms = kern_ms_total / max(1, kern_launches)
    sa_bytes = k1 * ncols * 8
    alg_bytes = bytes_step + sa_bytes                   # A read + SA write per launch
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()

    # ---- phase breakdown (untimed in the main line): cs_apply alone
    SA = synth.colmajor_empty(torch, k1, ncols, torch.float64, dev)
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        csk.cs_apply(plan, A, b=b, SA=SA)
    ev1.record(stream)
    barrier()
    cs_ms = ev0.elapsed_time(ev1) / args.steps
    ev0.record(stream)
    for _ in range(args.steps):
        csk.ms_apply(plan, k2, A, b=b, Z=Z)
    ev1.record(stream)
    barrier()
    msa_ms = ev0.elapsed_time(ev1) / args.steps
    t = time.perf_counter()
    for _ in range(0 if args.cs_only else args.steps):
        csk.ms_solve(Z, n, x=x)
    solve_ms = (time.perf_counter() - t) * 1e3 / args.steps

    # ---- SURVEY 8(d) "both input families" + the fp32 path: the CountSketch alone on kappa = 1e10 A
    # of the same shape (its speed must not depend on the values) and on the fp32 copy of [A b]
    families = None
    if ws == 1 and not args.no_extra and not args.cs_only and args.config in ("c2", "c3"):
        def time_cs(Ax, bx, SAx):
            for _ in range(2):
                csk.cs_apply(plan, Ax, b=bx, SA=SAx)
            barrier()
            ev0.record(stream)
            for _ in range(args.steps):
                csk.cs_apply(plan, Ax, b=bx, SA=SAx)
            ev1.record(stream)
            barrier()
            return ev0.elapsed_time(ev1) / args.steps

        families = {"gaussian_f64": {"ms": cs_ms, "gbs": bytes_step / (cs_ms * 1e-3) / 1e9}}
        buf2 = synth.colmajor_empty(torch, d, ncols, torch.float64, dev)
        buf2[:, :n] = synth.ill_conditioned_torch(d, n, 1e10, seed=DATA_SEED, device=dev)
        buf2[:, n] = b
        t_ill = time_cs(buf2[:, :n], buf2[:, n], SA)
        families["kappa1e10_f64"] = {"ms": t_ill, "gbs": bytes_step / (t_ill * 1e-3) / 1e9}
        del buf2
        buf32 = synth.colmajor_empty(torch, d, ncols, torch.float32, dev)
        buf32.copy_(buf)
        SA32 = synth.colmajor_empty(torch, k1, ncols, torch.float32, dev)
        t32 = time_cs(buf32[:, :n], buf32[:, n], SA32)
        families["gaussian_f32"] = {"ms": t32, "gbs": bytes_step / 2 / (t32 * 1e-3) / 1e9}
        del buf32, SA32
        torch.cuda.empty_cache()

    # ---- plan costs, warm (cuBLAS and the modules already loaded): codes (a1) of a second plan, and
    # the Gaussian G (a4) it draws on first use = its first ms_apply minus a warm ms_apply
    ev0.record(stream)
    plan2 = csk.cs_plan(d, k1, SKETCH_SEED + 1, row0=row0)
    ev1.record(stream)
    barrier()
    plan_warm_ms = ev0.elapsed_time(ev1)
    ev0.record(stream)
    csk.ms_apply(plan2, k2, A, b=b, Z=Z)
    ev1.record(stream)
    barrier()
    g_gen_ms = max(0.0, ev0.elapsed_time(ev1) - msa_ms)
    plan2.close()

    # ---- roofline attribution of the dominant kernel (N = 1): the same launch with its A loads
    # skipped (reduce path alone) and with its reductions skipped (HBM read path alone), via the
    # library's compile-time experiment variants (CSK_EXP, DESIGN.md 6.1/6.1b).  If the full
    # kernel runs at the reduce-only time, the L2 fp64 reduction rate -- not HBM -- bounds it.
    attribution = None
    if ws == 1 and not args.no_extra and args.variant in ("auto", "B"):
        def time_exp(e):
            os.environ["CSK_EXP"] = str(e)
            try:
                for _ in range(2):
                    csk.cs_apply(plan, A, b=b, SA=SA)
                barrier()
                ev0.record(stream)
                for _ in range(args.steps):
                    csk.cs_apply(plan, A, b=b, SA=SA)
                ev1.record(stream)
                barrier()
                return ev0.elapsed_time(ev1) / args.steps
            finally:
                del os.environ["CSK_EXP"]
        red_ms, load_ms = time_exp(2), time_exp(1)
        attribution = {"cs_apply_ms": cs_ms, "reduce_path_only_ms": red_ms, "load_path_only_ms": load_ms,
                       "load_path_gbs": bytes_step / (load_ms * 1e-3) / 1e9,
                       "kernel_over_reduce_path": kern_ms / red_ms,
                       "note": "reduce path alone = every row's bulk reduce-add into the L2-resident SA^T with the "
                               "A loads skipped; the kernel is bound by whichever path is slower"}

    # ---- the Count+SRHT multisketch step on the same [A b], for comparison
    msh = None
    if ws == 1 and not args.no_extra and not args.cs_only and (k1 & (k1 - 1)) == 0:
        Zh = synth.colmajor_empty(torch, k2, ncols, torch.float64, dev)
        def msh_step():
            csk.msh_apply(plan, k2, A, b=b, Z=Zh)
            csk.ms_solve(Zh, n, x=x)
        for _ in range(2):
            msh_step()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            msh_step()
        ev1.record(stream)
        barrier()
        msh = {"step_ms": ev0.elapsed_time(ev1) / args.steps,
               "rel_residual": float(torch.linalg.norm(b - A @ x) / torch.linalg.norm(b)),
               "what": "msh_apply (CountSketch + SRHT_k2 over the k1 sketch rows) + ms_solve"}
        del Zh

    # ---- normal-equations baseline (a8) on the same [A b]
    ne = {"gram": os.environ.get("CSK_NE_GRAM", "cuBLAS DGEMM A^T A + DGEMV A^T b + DDOT b^T b, one-CTA augmented Cholesky")}
    def ne_call():
        # the Gram + Cholesky work is done whether or not a pivot fails (ENOTPD is the
        # breakdown of Fig 8), so the time is recorded either way, with the status
        try:
            csk.ne_lstsq(A, b, x=x)
            return "OK"
        except csk.CskError as e:
            return str(e).split(":")[1].strip()

    if args.no_ne:
        ne.update(status="skipped (--no-ne)", ms=None)
    else:
        for _ in range(max(1, args.warmup // 2)):
            ne_call()
        barrier()
        ev0.record(stream)
        statuses = [ne_call() for _ in range(args.steps)]
        ev1.record(stream)
        barrier()
        ne["ms"] = ev0.elapsed_time(ev1) / args.steps
        ne["status"] = statuses[-1]

    # ---- accuracy of the step's solution (verification, untimed): ||b - A x|| / ||b||
    acc = {}
    if not args.cs_only:
        step()
        join()
        torch.cuda.synchronize()
        acc["rel_residual_ms"] = float(torch.linalg.norm(b - A @ x) / torch.linalg.norm(b))
    if ws == 1 and d * ncols * 8 <= 16e9 and not args.no_acc and not args.cs_only:
        R = torch.linalg.qr(buf, mode="r")[1]
        acc["rel_residual_true"] = float(abs(R[n, n]) / torch.linalg.norm(b))
        del R
        if ne["status"] == "OK":
            csk.ne_lstsq(A, b, x=x)
            acc["rel_residual_ne"] = float(torch.linalg.norm(b - A @ x) / torch.linalg.norm(b))

    # ---- e2e: C-ABI with HOST buffers (pinned), H2D inside the timed region
    e2e = None
    if not args.no_e2e:
        hbuf = torch.empty((ncols, d), dtype=torch.float64, pin_memory=True)
        hbuf.copy_(buf.t())
        hA, hb = hbuf.t()[:, :n], hbuf[n]
        hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
        csk.ms_lstsq(plan, k2, hA, hb, x=hx)           # warm
        ke = max(1, min(args.steps, 3))
        barrier()
        t = time.perf_counter()
        for _ in range(ke):
            csk.ms_lstsq(plan, k2, hA, hb, x=hx)
        barrier()
        e2e_ms = max_over_ranks((time.perf_counter() - t) * 1e3 / ke)
        e2e = {"value": ws * bytes_step / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": bytes_step, "d2h_bytes_per_step": n * 8 + 16, "steps": ke,
               "path": "ms_lstsq(host A, b, x): row chunks streamed H2D on a copy stream, overlapped with the sketch"}
        del hbuf

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        rows, _, _ = oracle_sample_rows(n, 15.0, k1, k2)
        rows = min(rows, d)
        tcpu = run_oracle_sample(cfg, rows)
        cpu = {"value": rows * ncols * 8 / tcpu / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"first {rows} rows (+b) of the workload shape, oracle ms_lstsq (codes, CountSketch, G, "
                         f"G-stage, Householder), {tcpu:.1f} s", "host_cores_available": cpu_cores()}

    variant = os.environ.get("CSK_VARIANT", "auto")
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "step_ms_stats": step_stats,
        "config": {"workload": cfg["name"], "d_per_rank": d, "d_global": d_glob, "n": n, "k1": k1, "k2": k2,
                   "rhs": "b = A e + eta, eta ~ N(0, 0.01)", "variant": variant,
                   "codes": "hashed on the fly" if args.hash_plan else "stored (4 B/row)",
                   "pipeline": ("solve of step i on a second stream, overlapping step i+1's sketch (Z, x "
                                "double-buffered)") if pipe else "serial (one stream)",
                   "l2": "inputs (%.1f GB per rank) > 126 MB L2; no flush needed" % (bytes_step / 1e9),
                   "parallelism": f"row-partitioned dp{ws}" + (f" + {backend.upper()} all-reduce of Z" if ws > 1 else "")},
        "clocks": clocks.summary(),
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.config, variant), "kernel": "cs_apply main kernel",
                     "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / step_ms,
                     "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                     "frac_of_8TBs_nominal": achieved / NOMINAL_HBM_GBS, "attribution": attribution},
        "cpu_baseline": cpu,
        "phases_ms": {"cs_apply": cs_ms, "g_stage": msa_ms - cs_ms, "solve": solve_ms,
                      "plan_codes_warm": plan_warm_ms, "g_generation_warm": g_gen_ms,
                      "plan_codes_first_call": plan_ms, "first_ms_apply_incl_library_init": gauss_first_ms},
        "cs_apply_gbs": bytes_step / (cs_ms * 1e-3) / 1e9,
        "cs_apply_input_families": families,
        "count_srht_multisketch": msh,
        "normal_equations": ne,
        "speedup_vs_ne": (ne["ms"] / step_ms) if ne.get("ms") else None,
        "accuracy": acc,
    }
    if ws == 1 and not args.no_ls and args.config == "c2":
        # the least-squares comparison on BASELINE.json's C4 ([A b], d=2^23, n=128, k1=32768,
        # k2=256): kappa = 1e10 (the BJ config: NE breaks down) and kappa = 1e2 (the
        # paper's timing setup: both solvers accurate -> matched-accuracy speedup)
        del buf, A, b, SA_ws, Z, x, SA
        torch.cuda.empty_cache()
        line["ls_c4"] = {f"kappa_{k:.0e}": ls_compare(args, CONFIGS["c4"], k, dev, stream) for k in (1e10, 1e2)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------- NEXT rows: SRHT and rand_cholQR
NEXT_CONFIGS = {
    "srht": dict(d=1 << 24, n=64, k=128,
                 name="NEXT-3 SRHT (P:L164-173) of [A b], d=2^24, n=64 (+b), k=2n=128, fp64 col-major, Gaussian A"),
    "rc": dict(d=1 << 23, n=128, k1=32768, k2=256, kappa=1e10,
               name="NEXT-1 rand_cholQR LS (Alg 5) on C4's [A b]: d=2^23, n=128, kappa(A)=1e10, k1=2n^2, k2=2n"),
}
NEXT_CONFIGS["kappa"] = dict(d=1 << 17, n=16,
                             name="NEXT-4 Fig 8 kappa sweep (P:L360-369): d=2^17, n=16, b = A e, kappa(A) = 1 .. 1e14")
NEXT_CONFIGS["fig35"] = dict(name="Figs 3-5 grid (P:L240-336): d in {2^21, 2^22, 2^23}, n in {32, 64, 128, 256}; "
                                   "sketch and least-squares times of every operator on one B200")
DGEMM_TFS_MEASURED = 35.41   # profiles/r01_measured_b200.json: cuBLAS DGEMM 8192^3 on this pool's B200


def _timed(fn, steps, warmup, stream):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def bench_kappa(args, cfg):
    """Fig 8 as a GPU experiment: relative residual ||b - Ax|| / ||b|| of every solver vs kappa(A) on
    a consistent b = A e (an exact solution exists).  NE degrades past kappa ~ 1e8; the
    sketch-and-solve solvers and rand_cholQR track the QR solve."""
    import torch
    import paper_2508_14209_b200 as csk
    import synth
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    d, n = cfg["d"], cfg["n"]
    k1, k2 = 2 * n * n, 2 * n
    plan = csk.cs_plan(d, k1, SKETCH_SEED)
    rows = []
    t0 = time.perf_counter()
    for e in range(0, 15, 2):
        kappa = 10.0 ** e
        A = synth.ill_conditioned_torch(d, n, kappa, seed=DATA_SEED, device=dev)
        b = synth.rhs_torch(A, "consistent", seed=DATA_SEED)
        nb = float(torch.linalg.norm(b))
        row = {"kappa": kappa}
        def resid(x):
            return float(torch.linalg.norm(b - A @ x)) / nb
        solvers = {
            "ne": lambda: csk.ne_lstsq(A, b),
            "ms": lambda: csk.ms_lstsq(plan, k2, A, b)[0],
            "msh": lambda: csk.msh_lstsq(plan, k2, A, b)[0],
            "cs": lambda: csk.cs_lstsq(plan, A, b)[0],
            "gs": lambda: csk.gs_lstsq(A, b, k2, SKETCH_SEED)[0],
            "rc": lambda: csk.rc_lstsq(plan, k2, A, b),
        }
        for name, fn in solvers.items():
            try:
                row[name] = resid(fn())
            except csk.CskError as ex:
                row[name] = str(ex).split(":")[1].strip()
        Q, R = torch.linalg.qr(A)
        row["qr"] = resid(torch.linalg.solve_triangular(R, (Q.t() @ b)[:, None], upper=True)[:, 0])
        rows.append(row)
    line = {"metric": "relative residual ||b - Ax||/||b|| vs kappa(A), b = A e (Fig 8)", "value": None,
            "unit": "ratio", "n_gpus": 1, "steps": 1, "warmup": 0, "ms_per_step": (time.perf_counter() - t0) * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "k1": k1, "k2": k2}, "sweep": rows,
            "note": "accuracy experiment (P:L360-369), not a throughput line; NE fails past kappa ~ 1e8"}
    print(json.dumps(line), flush=True)
    return 0


def bench_fig35(args, cfg):
    """The paper's evaluation grid on B200: per (d, n), sketch times (Fig 3: Gram A^T A, Gaussian sketch
    k = 2n, CountSketch k1 = 2n^2, SRHT k = 2n, multisketch 2n x 2n^2) with their HBM throughput
    (Fig 4: % of the measured copy bandwidth), and least-squares times (Fig 5: NE, Gaussian,
    CountSketch-only, multisketch, rand_cholQR; kappa(A) = 1e2 as in P:L322)."""
    import torch
    import paper_2508_14209_b200 as csk
    import synth
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    peak, _ = hbm_peak()
    steps, warm = max(3, args.steps // 4), 2
    grid = []
    t0 = time.perf_counter()
    for logd in (21, 22, 23):
        for n in (32, 64, 128, 256):
            d = 1 << logd
            k1, k2 = 2 * n * n, 2 * n
            buf = synth.colmajor_empty(torch, d, n + 1, torch.float64, dev)
            buf[:, :n] = synth.ill_conditioned_torch(d, n, 1e2, seed=DATA_SEED, device=dev)
            buf[:, n] = synth.rhs_torch(buf[:, :n], "easy", seed=DATA_SEED)
            A, b = buf[:, :n], buf[:, n]
            plan = csk.cs_plan(d, k1, SKETCH_SEED)
            x = torch.empty(n, dtype=torch.float64, device=dev)
            abytes = d * n * 8
            C = torch.empty((n, n), dtype=torch.float64, device=dev)
            t = {}
            t["gram"] = _timed(lambda: torch.matmul(A.t(), A, out=C), steps, warm, stream)
            t["gaussian"] = _timed(lambda: csk.gs_apply(A, k2, SKETCH_SEED), steps, warm, stream)
            t["countsketch"] = _timed(lambda: csk.cs_apply(plan, A), steps, warm, stream)
            t["srht"] = _timed(lambda: csk.srht_apply(A, k2, SKETCH_SEED), steps, warm, stream)
            t["multisketch"] = _timed(lambda: csk.ms_apply(plan, k2, A), steps, warm, stream)
            ls = {}
            def ne():
                try:
                    csk.ne_lstsq(A, b, x=x)
                except csk.CskError:
                    pass
            ls["ne"] = _timed(ne, steps, warm, stream)
            ls["gaussian"] = _timed(lambda: csk.gs_lstsq(A, b, k2, SKETCH_SEED, x=x), steps, warm, stream)
            ls["countsketch"] = _timed(lambda: csk.cs_lstsq(plan, A, b, x=x), steps, warm, stream)
            ls["multisketch"] = _timed(lambda: csk.ms_lstsq(plan, k2, A, b, x=x), steps, warm, stream)
            ls["rand_cholqr"] = _timed(lambda: csk.rc_lstsq(plan, k2, A, b, x=x), steps, warm, stream)
            grid.append({"d": d, "n": n, "sketch_ms": t, "lstsq_ms": ls,
                         "sketch_pct_of_hbm": {k: 100.0 * abytes / (v * 1e-3) / 1e9 / peak for k, v in t.items()},
                         "speedup_multisketch_vs_ne": ls["ne"] / ls["multisketch"]})
            log(f"[fig35] d=2^{logd} n={n}: " + ", ".join(f"{k} {v:.2f}" for k, v in ls.items()))
            del buf, A, b, plan, C
            torch.cuda.empty_cache()
    line = {"metric": "sketch and least-squares times over the paper's (d, n) grid (Figs 3-5)", "value": None,
            "unit": "ms", "n_gpus": 1, "steps": steps, "warmup": warm, "ms_per_step": (time.perf_counter() - t0) * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "kappa": 1e2, "rhs": "easy"}, "grid": grid,
            "note": "Gram = torch.matmul (cuBLAS DGEMM) A^T A; pct_of_hbm = d*n*8 bytes / time / measured copy BW"}
    print(json.dumps(line), flush=True)
    return 0


def bench_next(args, cfg):
    """One JSON line for a NEXT row, N = 1 (N > 1: rank 0 runs, the others exit; these rows are
    measured on one GPU).  Same contract keys as the main line."""
    import torch
    import paper_2508_14209_b200 as csk
    import synth
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    d, n = cfg["d"], cfg["n"]
    ncols = n + 1
    buf = synth.colmajor_empty(torch, d, ncols, torch.float64, dev)
    if args.config == "rc":
        buf[:, :n] = synth.ill_conditioned_torch(d, n, cfg["kappa"], seed=DATA_SEED, device=dev)
        buf[:, n] = synth.rhs_torch(buf[:, :n], "easy", seed=DATA_SEED)
    else:
        buf.copy_(synth.gaussian_matrix_torch(d, ncols, seed=DATA_SEED, device=dev))
    A, b = buf[:, :n], buf[:, n]
    nbytes = d * ncols * 8
    peak, peak_src = hbm_peak()
    csk.launch_count(reset=True)
    if args.config == "srht":
        k = cfg["k"]
        Y = torch.empty((ncols, k), dtype=torch.float64, device=dev).t()
        step = lambda: csk.srht_apply(A, k, SKETCH_SEED, b=b, Y=Y)   # noqa: E731
        for _ in range(args.warmup):
            step()
        launches0 = csk.launch_count(reset=True)
        with ClockSampler(local) as clocks:
            csk.profile_enable(True)
            ms = _timed(step, args.steps, 0, stream)
            kms, kl = csk.profile_read()
            csk.profile_enable(False)
        launches = csk.launch_count() // max(1, args.steps)
        kern_ms = kms / max(1, kl)
        achieved = nbytes / (kern_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "kernel": "srht_warp_kernel", "kernel_ms": kern_ms,
                "kernel_share_of_step": kern_ms / ms, "alg_bytes_per_launch": nbytes, "peak_source": peak_src,
                "note": "algorithmic bytes = d*(n+1)*8 (A and b read once; D bits d/8 B and Y k*(n+1)*8 B not counted)"}
        # e2e: host [A b] -> device -> SRHT -> Y back to the host
        hbuf = torch.empty((ncols, d), dtype=torch.float64).pin_memory().t()
        hbuf.copy_(buf)
        hY = torch.empty((ncols, k), dtype=torch.float64).pin_memory().t()
        def e2e_step():
            buf.copy_(hbuf, non_blocking=True)
            csk.srht_apply(A, k, SKETCH_SEED, b=b, Y=Y)
            hY.copy_(Y, non_blocking=True)
        e2e_ms = _timed(e2e_step, 3, 1, stream)
        e2e = {"value": nbytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": k * ncols * 8, "ms_per_step": e2e_ms}
        # the oracle on a bounded sample (2^16 rows of the same shape)
        import oracle
        rows = 1 << 16
        sample = buf[:rows].cpu().numpy()
        t = time.perf_counter()
        oracle.srht_apply(sample[:, :n], k, SKETCH_SEED, b=sample[:, n])
        tcpu = time.perf_counter() - t
        cpu = {"value": rows * ncols * 8 / tcpu / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"first {rows} rows of the workload (d=2^16 SRHT, radix-4 FWHT per column), {tcpu:.2f} s"}
        value, unit, metric = nbytes / (ms * 1e-3) / 1e9, "GB/s", "SRHT apply GB/s (% HBM peak)"
        extra = {}
    else:
        k1, k2 = cfg["k1"], cfg["k2"]
        plan = csk.cs_plan(d, k1, SKETCH_SEED)
        x = torch.empty(n, dtype=torch.float64, device=dev)
        step = lambda: csk.rc_lstsq(plan, k2, A, b, x=x)   # noqa: E731
        for _ in range(args.warmup):
            step()
        csk.launch_count(reset=True)
        with ClockSampler(local) as clocks:
            ms = _timed(step, args.steps, 0, stream)
        launches = csk.launch_count() // max(1, args.steps)
        # the dominant kernel: the fused TRSM + Gram pass (rc_gram), timed alone on the same inputs
        Z = csk.ms_apply(plan, k2, A, b=b)
        R0 = csk.rc_r0(Z, n)
        gram_ms = _timed(lambda: csk.rc_gram(A, b, R0), args.steps, 2, stream)
        flops = 2.0 * d * n * n        # TRSM d n^2 + SYRK-form Gram d n^2
        achieved = flops / (gram_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": DGEMM_TFS_MEASURED, "unit": "TFLOP/s",
                "frac": achieved / DGEMM_TFS_MEASURED, "traffic": None, "kernel": "rc_pass_ws_kernel (rc_gram)",
                "kernel_ms": gram_ms, "kernel_share_of_step": gram_ms / ms,
                "alg_flops_per_launch": flops,
                "peak_source": "fp64 DMMA: measured cuBLAS DGEMM 8192^3 (profiles/r01_measured_b200.json); "
                               "MEASURED_PEAKS.json has no fp64 figure"}
        rel = float(torch.linalg.norm(b - A @ x) / torch.linalg.norm(b))
        Rq = torch.linalg.qr(buf, mode="r")[1]
        extra = {"rel_residual": rel, "true_rel_residual": float(abs(Rq[n, n]) / torch.linalg.norm(b))}
        del Rq
        try:
            ne_ms = _timed(lambda: csk.ne_lstsq(A, b, x=x), args.steps, 1, stream)
            extra["ne_ms"], extra["ne_status"] = ne_ms, "OK"
        except csk.CskError as e:
            extra["ne_status"] = str(e).split(":")[1].strip()
        e2e, cpu = None, None
        value, unit, metric = nbytes / (ms * 1e-3) / 1e9, "GB/s", "rand_cholQR LS: [A b] GB/s through rc_lstsq"
        extra["ms_lstsq_distortion_free"] = True
    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["name"], "l2": "inputs > 126 MB L2; no flush needed"},
            "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu}
    line.update(extra)
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS) + sorted(NEXT_CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="auto", choices=["auto", "L", "T", "S", "G", "B", "X"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pipeline", action="store_true", help="(default) step i's solve on a second stream, "
                                                                "overlapping step i+1's sketch (DESIGN.md 7)")
    ap.add_argument("--no-pipeline", action="store_true", help="one stream per step (serial)")
    ap.add_argument("--hash-plan", action="store_true",
                    help="CSK_PLAN_HASH: no stored codes, the CountSketch kernel hashes rows on the fly")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ne", action="store_true", help="skip the normal-equations baseline")
    ap.add_argument("--cs-only", action="store_true", help="experiment mode: a step is cs_apply alone")
    ap.add_argument("--no-acc", action="store_true", help="skip the untimed accuracy checks")
    ap.add_argument("--no-ls", action="store_true", help="skip the C4 least-squares comparison (N=1, c2)")
    ap.add_argument("--no-extra", action="store_true", help="skip the kappa=1e10 / fp32 CountSketch lines")
    ap.add_argument("--no-ls-extra", action="store_true",
                    help="LS comparison without the Gaussian / CountSketch-only / Count+SRHT solvers")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.config in NEXT_CONFIGS:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "NEXT rows are measured against the oracle inside "
                                                                  "the line's cpu_baseline"}))
            return 0
        if args.config == "kappa":
            return bench_kappa(args, NEXT_CONFIGS["kappa"])
        if args.config == "fig35":
            return bench_fig35(args, NEXT_CONFIGS["fig35"])
        return bench_next(args, NEXT_CONFIGS[args.config])
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return bench_reference(args, cfg)
    return bench_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
