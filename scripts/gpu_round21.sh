#!/bin/bash
set -u
TAG=${1:-r02c}
mkdir -p gpurun_out
timeout 300 python scripts/factor_profile.py sketch > gpurun_out/${TAG}_factor_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/${TAG}_factor_plain.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_factor_launches.csv python scripts/factor_profile.py sketch > gpurun_out/${TAG}_factor_ncu.log 2>&1; echo "ncu rc=$?"
