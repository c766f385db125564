#!/bin/bash
# CPQR L2 batching A/B: compression time per level (trace) and build digests
set -u
for f in 0 0.5 0.35 0.7; do
  echo "== SVMHSS_CPQR_L2FRAC=$f"
  for smp in sketch ann; do
    SVMHSS_CPQR_L2FRAC=$f SVMHSS_TRACE=1 timeout 400 python scripts/cpqr_ab.py 2 $smp > /tmp/t.log 2>&1
    grep mode= /tmp/t.log | cut -c1-120
    awk '/trace\] hss_compress/{c++} c==2' /tmp/t.log | grep "cpqr" | awk '{print $3}' | paste -sd' '
  done
done
