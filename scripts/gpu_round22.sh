#!/bin/bash
# source-level ncu of the single-node QR / Cholesky / larft launches of the factor
set -u
TAG=${1:-r02d}
mkdir -p gpurun_out
timeout 300 python scripts/factor_profile.py ann > gpurun_out/${TAG}_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"${KRE:-bgeqrf|bpotrf|blarft}" --launch-skip ${SKIP:-27} -c ${CNT:-6} -o gpurun_out/${TAG}_small python scripts/factor_profile.py ann > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
