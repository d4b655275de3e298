#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cs_apply or partition or ms_apply or hash" 2>&1 | tail -2
for r in 1 2; do for lib in "" scratch_ab/libcsk_prev.so; do CSK_LIB_OVERRIDE=$lib timeout 300 python scripts/f32_once.py; done; done
