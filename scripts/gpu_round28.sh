#!/bin/bash
# forward-sweep A/B: chunk rows per CTA and L2 prefetch (ADMM loop ms/iteration, 200 iterations)
set -u
for rep in 1 2; do
  for cfg in "32 0" "64 0" "32 1" "64 1" "16 0"; do
    set -- $cfg
    echo -n "ch=$1 prefetch=$2: "; SVMHSS_FWD_CH=$1 SVMHSS_FWD_PREFETCH=$2 timeout 300 python scripts/admm_profile.py 2>&1 | grep loop
  done
done
