#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "narrow_rows or cs_apply_fp64" 2>&1 | tail -n 2
cat > gpurun_out/mix.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2508_14209_b200 as csk, synth
for logd, n in ((23, 32), (22, 32), (23, 16)):
    d = 1 << logd
    A = synth.gaussian_matrix_torch(d, n, seed=2)
    plan = csk.cs_plan(d, 2 * n * n, 1)
    SA = torch.empty((n, 2 * n * n), dtype=torch.float64, device="cuda").t()
    for _ in range(3): csk.cs_apply(plan, A, SA=SA)
    torch.cuda.synchronize()
    csk.profile_enable(True)
    for _ in range(10): csk.cs_apply(plan, A, SA=SA)
    ms, k = csk.profile_read(); csk.profile_enable(False)
    print(f"mix_rt={os.environ.get('CSK_MIX_RT','16')} d=2^{logd} n={n}: {ms/k:.4f} ms, {d*n*8/(ms/k*1e-3)/1e9:.0f} GB/s")
PY
for rt in 32 24 16 8 0; do CSK_MIX_RT=$rt timeout 300 python gpurun_out/mix.py; done
