#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
for cv in "" 100 50; do
  echo "carve=$cv"; CSK_SRHT_CARVE=$cv timeout 300 python scripts/srht_once.py; CSK_SRHT_CARVE=$cv N=64 LOGD=24 timeout 300 python scripts/srht_once.py
done
done
CSK_SRHT_KERNEL=2 timeout 300 python scripts/srht_once.py
