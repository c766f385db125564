#!/bin/bash
set -u
for pf in 1 0 1; do
  echo "== SVMHSS_CPQR_PREFETCH=$pf"
  for smp in sketch ann; do
    SVMHSS_CPQR_PREFETCH=$pf SVMHSS_TRACE=1 timeout 400 python scripts/cpqr_ab.py 2 $smp > /tmp/t.log 2>&1
    grep mode= /tmp/t.log | cut -c1-100
    awk '/trace\] hss_compress/{c++} c==2' /tmp/t.log | grep "cpqr" | awk '{print $3}' | paste -sd' '
  done
done
