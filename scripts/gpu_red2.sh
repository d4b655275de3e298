#!/bin/bash
# C2 reduce-path attribution: EXP=2 (no A loads) at full / half grid; SA^T row padding (CSK_LC)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {
  env "$@" timeout 600 python bench.py --config ${CFG:-c2} --cs-only --no-cpu --no-e2e --no-ne --no-acc --no-ls --no-extra --steps 10 > gpurun_out/x.json 2> gpurun_out/x.err
  python -c "import json; d=json.load(open('gpurun_out/x.json')); r=d['roofline']; print('$*', 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))" || tail -n 3 gpurun_out/x.err
}
run CSK_X=0
run CSK_EXP=2
run CSK_EXP=2 CSK_GRID=74
run CSK_EXP=2 CSK_GRID=37
run CSK_EXP=1
run CSK_EXP=1 CSK_GRID=74
run CSK_LC=72
run CSK_LC=80
run CSK_LC=96
run CSK_LC=128
run CSK_EXP=2 CSK_LC=80
