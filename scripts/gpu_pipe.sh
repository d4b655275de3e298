#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in c2 c4; do
  CFG=$c timeout 300 python scripts/pipeline_exp.py
  for g in 140 132 124; do CFG=$c CSK_GRID=$g timeout 300 python scripts/pipeline_exp.py; done
done
