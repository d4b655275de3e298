#!/bin/bash
# B32 tile-row shift (bank-conflict-free STS): parity subset, then same-box A/B vs the previous library
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cs_apply or hash or partition or ms_apply or split or narrow or codes or sort" 2>&1 | tail -2
bash scripts/gpu_ab.sh
timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum --clock-control none -k regex:cs_bulk32 -c 1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-ne --no-acc --no-ls --no-extra --cs-only 2>&1 | grep -E "bank_conflicts|wavefronts|gpu__time"
