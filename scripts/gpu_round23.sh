#!/bin/bash
# tensor-core QR: parity suite + factor timing (+ launch list)
set -u
TAG=${1:-r02e}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
for smp in sketch ann; do
  timeout 300 python scripts/factor_profile.py $smp > gpurun_out/${TAG}_factor_$smp.log 2>&1; echo "factor $smp rc=$?"; tail -1 gpurun_out/${TAG}_factor_$smp.log
done
SVMHSS_QR_TC=0 timeout 300 python scripts/factor_profile.py sketch 2>&1 | tail -1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_factor_launches.csv python scripts/factor_profile.py sketch > gpurun_out/${TAG}_factor_ncu.log 2>&1; echo "ncu rc=$?"
