#!/bin/bash
# GEMM tile A/B on the factor (wall time, 3 reps each)
set -u
TAG=${1:-r02j}
mkdir -p gpurun_out
for v in 84 44 82 84 44; do
  echo -n "tile=$v "; SVMHSS_GEMM_TILE=$v timeout 300 python scripts/factor_profile.py sketch 2>&1 | tail -1
done
SVMHSS_GEMM_TILE=44 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_factor_launches.csv python scripts/factor_profile.py sketch > gpurun_out/${TAG}_factor_ncu.log 2>&1; echo "ncu rc=$?"
