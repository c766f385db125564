#!/bin/bash
# forward-sweep load-pattern A/B (ADMM loop ms/iteration, 200 iterations); results identical across modes
set -u
for rep in 1 2; do
  for m in 1 2 3 4 0; do
    echo -n "mode=$m: "; SVMHSS_FWD_MODE=$m timeout 300 python scripts/admm_profile.py 2>&1 | grep loop
  done
done
