#!/bin/bash
# persisting-L2 top levels A/B (ADMM loop ms/iteration, 200 iterations)
set -u
for rep in 1 2; do
  for mb in 0 48 100 20; do
    echo -n "persist_mb=$mb: "; SVMHSS_L2_PERSIST_MB=$mb timeout 300 python scripts/admm_profile.py 2>&1 | grep loop
  done
done
